"""Dev: fp32 (3xTF32) GEMM error vs fp64 as a function of K (chunk from GM_TF32_CHUNK)."""
import ctypes, os, sys
import torch
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
from paper_1611_07819_b200 import _lib as L
lib = L.load()
for k in (2048, 8192, 16384, 32768):
    m = n = 512
    g = torch.Generator(device="cuda").manual_seed(k)
    A = (torch.rand(m, k, device="cuda", generator=g, dtype=torch.float64) * 2 - 1).float()
    B = (torch.rand(k, n, device="cuda", generator=g, dtype=torch.float64) * 2 - 1).float()
    C = torch.zeros(m, n, device="cuda")
    errs = []
    for math in (0, 1):
        d = L.gm_gemm_desc(m=m, n=n, k=k, lda=k, ldb=n, ldc=n, trans_a=0, trans_b=0, prec_a=1, prec_b=1, prec_c=1,
                           math=math, cta_group=0, max_ctas=0, alpha=1.0, beta=0.0)
        ws = ctypes.c_uint64(); L.check(lib.gm_gemm_workspace_size(ctypes.byref(d), ctypes.byref(ws)))
        W = torch.empty(ws.value + 16, dtype=torch.uint8, device="cuda")
        L.check(lib.gm_gemm_local(ctypes.byref(d), A.data_ptr(), B.data_ptr(), C.data_ptr(), W.data_ptr(), ws.value, None))
        torch.cuda.synchronize()
        ref = A.double() @ B.double()
        errs.append(((C.double() - ref).norm() / ref.norm()).item())
    # plain fp32 sequential-ish reference error (cuBLAS fp32 SIMT) for context
    torch.backends.cuda.matmul.allow_tf32 = False
    e32 = (((A @ B).double() - ref).norm() / ref.norm()).item()
    print(f"chunk={os.environ.get('GM_TF32_CHUNK','256')} k={k} 3xtf32={errs[0]:.3e} 1xtf32={errs[1]:.3e} cublas_fp32={e32:.3e}", flush=True)
