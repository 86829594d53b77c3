# SPDX-License-Identifier: Apache-2.0
"""One local bf16 GEMM m x n x k (gm_gemm_local) repeated `reps` times, for
ncu captures of a single shape: python tools/dev/dev_one_gemm.py m n k reps"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
from paper_1611_07819_b200 import _lib as L  # noqa: E402

m, n, k = (int(x) for x in sys.argv[1:4])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
tb = int(sys.argv[5]) if len(sys.argv) > 5 else 0  # 1: B stored n x k (K-major)
lib = ctypes.CDLL(L.LIB_PATH)
lib.gm_gemm_local.argtypes = [ctypes.POINTER(L.gm_gemm_desc)] + [ctypes.c_void_p] * 4 + [ctypes.c_uint64, ctypes.c_void_p]
A = torch.randn(m, k, device="cuda").to(torch.bfloat16)
B = torch.randn(n, k, device="cuda").to(torch.bfloat16) if tb else torch.randn(k, n, device="cuda").to(torch.bfloat16)
C = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
d = L.gm_gemm_desc(m=m, n=n, k=k, lda=k, ldb=k if tb else n, ldc=n, trans_a=0, trans_b=tb, prec_a=3, prec_b=3, prec_c=3,
                   math=0, cta_group=2, max_ctas=0, alpha=1.0, beta=0.0)
st = torch.cuda.current_stream().cuda_stream
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for i in range(reps):
    if i == reps // 2:
        e0.record()
    assert lib.gm_gemm_local(ctypes.byref(d), A.data_ptr(), B.data_ptr(), C.data_ptr(), None, 0, st) == 0
e1.record()
torch.cuda.synchronize()
t = e0.elapsed_time(e1) / (reps - reps // 2)
print(f"ok m={m} n={n} k={k} transB={tb}: {t * 1e3:.1f} us {2 * m * n * k / t / 1e9:.1f} TFLOP/s")
