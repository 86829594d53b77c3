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
lib = ctypes.CDLL(L.LIB_PATH)
lib.gm_gemm_local.argtypes = [ctypes.POINTER(L.gm_gemm_desc)] + [ctypes.c_void_p] * 4 + [ctypes.c_uint64, ctypes.c_void_p]
A = torch.randn(m, k, device="cuda").to(torch.bfloat16)
B = torch.randn(k, n, device="cuda").to(torch.bfloat16)
C = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
d = L.gm_gemm_desc(m=m, n=n, k=k, lda=k, ldb=n, ldc=n, trans_a=0, trans_b=0, prec_a=3, prec_b=3, prec_c=3,
                   math=0, cta_group=2, max_ctas=0, alpha=1.0, beta=0.0)
st = torch.cuda.current_stream().cuda_stream
for _ in range(reps):
    assert lib.gm_gemm_local(ctypes.byref(d), A.data_ptr(), B.data_ptr(), C.data_ptr(), None, 0, st) == 0
torch.cuda.synchronize()
print("ok")
