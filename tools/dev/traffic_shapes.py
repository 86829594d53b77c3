# SPDX-License-Identifier: Apache-2.0
"""Dev harness for ncu: the per-GPU local GEMM launches of the bf16 32768^3
bench at N = 2 / 4 / 8 (2D grids 1x2, 2x2, 2x4; S = 2 row chunks per op), run
on one GPU with the same operand pitches the runtime uses (A band ld = k,
B from the band or the local tile, C tile pitch). Usage:
    python tools/dev/traffic_shapes.py N [reps]"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
from paper_1611_07819_b200 import _lib as L  # noqa: E402

SHAPES = {  # N -> (chunk rows m, tile cols n, k)
    2: (16384, 16384, 32768),
    4: (8192, 16384, 32768),
    8: (8192, 8192, 32768),
}


def main():
    world = int(sys.argv[1])
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    m, n, k = SHAPES[world]
    lib = ctypes.CDLL(L.LIB_PATH)
    lib.gm_gemm_local.argtypes = [ctypes.POINTER(L.gm_gemm_desc)] + [ctypes.c_void_p] * 4 + [ctypes.c_uint64,
                                                                                              ctypes.c_void_p]
    A = (torch.rand(2 * m, k, device="cuda") * 2 - 1).to(torch.bfloat16)  # the whole band: 2 chunks
    B = (torch.rand(k, n, device="cuda") * 2 - 1).to(torch.bfloat16)
    C = torch.empty(2 * m, n, device="cuda", dtype=torch.bfloat16)
    st = torch.cuda.current_stream().cuda_stream
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for rep in range(reps):
        if rep == reps - 1:
            start.record()
        for j in range(2):
            d = L.gm_gemm_desc(m=m, n=n, k=k, lda=k, ldb=n, ldc=n, trans_a=0, trans_b=0, prec_a=3, prec_b=3,
                               prec_c=3, math=0, cta_group=2, max_ctas=0, alpha=1.0, beta=0.0)
            rc = lib.gm_gemm_local(ctypes.byref(d), A.data_ptr() + j * m * k * 2, B.data_ptr(),
                                   C.data_ptr() + j * m * n * 2, None, 0, st)
            assert rc == 0
    end.record()
    torch.cuda.synchronize()
    ms = start.elapsed_time(end)
    print(f"N={world} op = 2 x {m}x{n}x{k}: {ms:.3f} ms, {2 * 2.0 * m * n * k / ms / 1e9:.1f} TFLOP/s", flush=True)


if __name__ == "__main__":
    main()
