"""Dev: Single-compute GEMM throughput (3xTF32 default, 1xTF32 opt-in) vs
cuBLAS fp32 (SIMT, allow_tf32 off) and cuBLAS TF32, device-timed."""
import ctypes, os, sys
import torch
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
from paper_1611_07819_b200 import _lib as L
lib = L.load()
for n in (int(a) for a in (sys.argv[1:] or ["8192", "16384"])):
    A = torch.rand(n, n, device="cuda") * 2 - 1
    B = torch.rand(n, n, device="cuda") * 2 - 1
    C = torch.empty(n, n, device="cuda")
    R = torch.empty(n, n, device="cuda", dtype=torch.float64)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    def timeit(fn, reps=3):
        fn(); torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            fn()
        e1.record(); torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps
    torch.matmul(A.double(), B.double(), out=R)
    for math in (0, 1):
        d = L.gm_gemm_desc(m=n, n=n, k=n, lda=n, ldb=n, ldc=n, trans_a=0, trans_b=0, prec_a=1, prec_b=1, prec_c=1,
                           math=math, cta_group=0, max_ctas=0, alpha=1.0, beta=0.0)
        ws = ctypes.c_uint64(); L.check(lib.gm_gemm_workspace_size(ctypes.byref(d), ctypes.byref(ws)))
        W = torch.empty(max(ws.value, 16), dtype=torch.uint8, device="cuda")
        st = torch.cuda.current_stream().cuda_stream
        ms = timeit(lambda: L.check(lib.gm_gemm_local(ctypes.byref(d), A.data_ptr(), B.data_ptr(), C.data_ptr(),
                                                      W.data_ptr(), ws.value, st)))
        err = float((C.double() - R).norm() / R.norm())
        print(f"ours {'3xTF32' if math == 0 else '1xTF32'} n={n}: {ms:.2f} ms {2*n**3/ms/1e9:.1f} TFLOP/s rel_fro {err:.2e}", flush=True)
    for tf32 in (False, True):
        torch.backends.cuda.matmul.allow_tf32 = tf32
        ms = timeit(lambda: torch.matmul(A, B, out=C))
        err = float((C.double() - R).norm() / R.norm())
        print(f"cuBLAS {'TF32' if tf32 else 'fp32'} n={n}: {ms:.2f} ms {2*n**3/ms/1e9:.1f} TFLOP/s rel_fro {err:.2e}", flush=True)
