# SPDX-License-Identifier: Apache-2.0
"""Config 2 (bf16 8192^3, one GPU) analysis in one process: our GEMM
(gm_gemm_local) and cuBLAS (torch.matmul) at M = N = 8192 over K, timed back
to back with CUDA events (50 reps, median of 5 batches), interleaved so both
see the same clock. A linear fit t(K) = fixed + K * slope separates the
per-launch fixed cost from the k-loop rate.
    python tools/dev/dev_c2_sweep.py"""
import ctypes
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
from paper_1611_07819_b200 import _lib as L  # noqa: E402

lib = ctypes.CDLL(L.LIB_PATH)
lib.gm_gemm_local.argtypes = [ctypes.POINTER(L.gm_gemm_desc)] + [ctypes.c_void_p] * 4 + [ctypes.c_uint64, ctypes.c_void_p]


def ours(A, B, C, m, n, k):
    d = L.gm_gemm_desc(m=m, n=n, k=k, lda=k, ldb=n, ldc=n, trans_a=0, trans_b=0, prec_a=3, prec_b=3, prec_c=3,
                       math=0, cta_group=2, max_ctas=0, alpha=1.0, beta=0.0)
    st = torch.cuda.current_stream().cuda_stream
    return lambda: lib.gm_gemm_local(ctypes.byref(d), A.data_ptr(), B.data_ptr(), C.data_ptr(), None, 0, st)


def timed(fn, reps=50):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    m = n = 8192
    ks = [1024, 2048, 4096, 8192, 16384]
    res = {("ours", k): [] for k in ks}
    res.update({("cublas", k): [] for k in ks})
    bufs = {}
    for k in ks:
        A = torch.randn(m, k, device="cuda").to(torch.bfloat16)
        B = torch.randn(k, n, device="cuda").to(torch.bfloat16)
        C = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
        bufs[k] = (A, B, C)
    for _ in range(5):
        for k in ks:
            A, B, C = bufs[k]
            res[("ours", k)].append(timed(ours(A, B, C, m, n, k)))
            res[("cublas", k)].append(timed(lambda: torch.matmul(A, B, out=C)))
    for who in ("ours", "cublas"):
        ts = [statistics.median(res[(who, k)]) for k in ks]
        # least squares t = a + b k
        kb = sum(ks) / len(ks)
        tb = sum(ts) / len(ts)
        b = sum((k - kb) * (t - tb) for k, t in zip(ks, ts)) / sum((k - kb) ** 2 for k in ks)
        a = tb - b * kb
        line = " ".join(f"K={k}: {t * 1e3:7.1f} us {2 * m * n * k / t / 1e9:7.1f} TF" for k, t in zip(ks, ts))
        print(f"{who:6s} {line}")
        print(f"{who:6s} fit: fixed {a * 1e3:6.1f} us + {b * 1e6:7.3f} ns per k  "
              f"(marginal {2 * m * n / b / 1e9:7.1f} TF)")


if __name__ == "__main__":
    main()
