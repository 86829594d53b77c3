"""Dev: cuBLAS DGEMM vs gm_gemm_local fp64 (DMMA) at n^3 (GM_F64_TILE picks the variant)."""
import ctypes, os, sys
import torch
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
from paper_1611_07819_b200 import _lib as L
lib = L.load()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
A = torch.randn(n, n, device="cuda", dtype=torch.float64); B = torch.randn(n, n, device="cuda", dtype=torch.float64)
C = torch.empty(n, n, device="cuda", dtype=torch.float64)
R = torch.empty(n, n, device="cuda", dtype=torch.float64)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
d = L.gm_gemm_desc(m=n, n=n, k=n, lda=n, ldb=n, ldc=n, trans_a=0, trans_b=0, prec_a=2, prec_b=2, prec_c=2, math=0, cta_group=0, max_ctas=0, alpha=1.0, beta=0.0)
for name, fn in (("cublas", lambda: torch.matmul(A, B, out=R)),
                 ("dmma", lambda: L.check(lib.gm_gemm_local(ctypes.byref(d), A.data_ptr(), B.data_ptr(), C.data_ptr(), None, 0, torch.cuda.current_stream().cuda_stream)))):
    fn(); torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{name} variant={os.environ.get('GM_F64_TILE', '64')} fp64 n={n}: {ms:.2f} ms {2*n**3/ms/1e9:.1f} TFLOP/s", flush=True)
print(f"rel_fro(dmma, cublas) = {float(torch.linalg.norm(C - R) / torch.linalg.norm(R)):.3e}")
