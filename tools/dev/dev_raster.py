"""Dev: one bf16 GEMM n^3 through gm_gemm_local (for ncu raster/traffic sweeps)."""
import ctypes, os, sys
import torch
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
from paper_1611_07819_b200 import _lib as L
lib = L.load()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
pad = int(sys.argv[3]) if len(sys.argv) > 3 else 0
A = torch.randn(n, n + pad, device="cuda", dtype=torch.bfloat16); B = torch.randn(n, n + pad, device="cuda", dtype=torch.bfloat16)
C = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
d = L.gm_gemm_desc(m=n, n=n, k=n, lda=n + pad, ldb=n + pad, ldc=n, trans_a=0, trans_b=0, prec_a=3, prec_b=3, prec_c=3, math=0,
                   cta_group=0, max_ctas=0, alpha=1.0, beta=0.0)
st = torch.cuda.current_stream().cuda_stream
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for i in range(reps):
    e0.record(); L.check(lib.gm_gemm_local(ctypes.byref(d), A.data_ptr(), B.data_ptr(), C.data_ptr(), None, 0, st)); e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
cs = int(C.view(torch.int16).to(torch.int64).sum().item())
med = sorted(ts[reps // 3:])[len(ts[reps // 3:]) // 2]
print(f"chunks={os.environ.get("GM_TC_CHUNKS","auto")} sync={os.environ.get("GM_TC_SYNC","auto")} group={os.environ.get("GM_RASTER_GROUP","16")} n={n} median {med:.3f} ms {2*n**3/med/1e9:.1f} TFLOP/s (last {ts[-1]:.3f}) die={os.environ.get('GM_DIE_AWARE','0')} checksum={cs}")
