for rep in 1 2; do
  python tools/dev/dev_raster.py 8192 40
  GM_NO_TMA_STORE=1 python tools/dev/dev_raster.py 8192 40
  GM_TC_SYNC=0 python tools/dev/dev_raster.py 8192 40
done > gpurun_out/sweep8192e.txt 2>&1
for K in 4096 8192 16384 32768; do python - <<PY >> gpurun_out/sweep8192e.txt 2>&1
import ctypes, os, sys, torch
sys.path.insert(0, ".")
from paper_1611_07819_b200 import _lib as L
lib = L.load()
m = n = 8192; k = $K
A = torch.randn(m, k, device="cuda", dtype=torch.bfloat16); B = torch.randn(k, n, device="cuda", dtype=torch.bfloat16)
C = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
d = L.gm_gemm_desc(m=m, n=n, k=k, lda=k, ldb=n, ldc=n, trans_a=0, trans_b=0, prec_a=3, prec_b=3, prec_c=3, math=0, cta_group=0, max_ctas=0, alpha=1.0, beta=0.0)
st = torch.cuda.current_stream().cuda_stream
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(5): L.check(lib.gm_gemm_local(ctypes.byref(d), A.data_ptr(), B.data_ptr(), C.data_ptr(), None, 0, st))
torch.cuda.synchronize(); e0.record()
for _ in range(20): L.check(lib.gm_gemm_local(ctypes.byref(d), A.data_ptr(), B.data_ptr(), C.data_ptr(), None, 0, st))
e1.record(); torch.cuda.synchronize(); ms = e0.elapsed_time(e1) / 20
print(f"8192x8192xk={k}: {ms*1e3:.1f} us {2*m*n*k/ms/1e9:.1f} TFLOP/s", flush=True)
PY
done
