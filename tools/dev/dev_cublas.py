"""Dev: torch.matmul (cuBLAS) bf16 n^3 for ncu comparison."""
import sys, torch
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
A = torch.randn(n, n, device="cuda", dtype=torch.bfloat16); B = torch.randn(n, n, device="cuda", dtype=torch.bfloat16)
C = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for i in range(int(sys.argv[2]) if len(sys.argv) > 2 else 4):
    e0.record(); torch.matmul(A, B, out=C); e1.record(); torch.cuda.synchronize()
print(f"cublas n={n} {e0.elapsed_time(e1):.3f} ms {2*n**3/e0.elapsed_time(e1)/1e9:.1f} TFLOP/s")
