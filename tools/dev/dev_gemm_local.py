"""Dev harness: gm_gemm_local vs a torch float64 reference on one GPU."""
import ctypes, sys, time
import torch
sys.path.insert(0, __import__("os").path.join(__import__("os").path.dirname(__file__), "..", ".."))
from paper_1611_07819_b200 import _lib as L

lib = ctypes.CDLL(L.LIB_PATH)
lib.gm_gemm_local.argtypes = [ctypes.POINTER(L.gm_gemm_desc)] + [ctypes.c_void_p] * 4 + [ctypes.c_uint64, ctypes.c_void_p]
lib.gm_gemm_workspace_size.argtypes = [ctypes.POINTER(L.gm_gemm_desc), ctypes.POINTER(ctypes.c_uint64)]
lib.gm_last_error.restype = ctypes.c_char_p
TD = {0: torch.float16, 1: torch.float32, 2: torch.float64, 3: torch.bfloat16}

def run(m, n, k, ta, tb, pa, pb, pc, cg, math=0, alpha=1.0, beta=0.0, ws_cache={}):
    g = torch.Generator(device="cuda").manual_seed(m * 7 + n * 13 + k)
    A = (torch.rand((k, m) if ta else (m, k), device="cuda", generator=g, dtype=torch.float64) * 2 - 1).to(TD[pa])
    B = (torch.rand((n, k) if tb else (k, n), device="cuda", generator=g, dtype=torch.float64) * 2 - 1).to(TD[pb])
    C = (torch.rand((m, n), device="cuda", generator=g, dtype=torch.float64) * 2 - 1).to(TD[pc])
    C0 = C.clone()
    d = L.gm_gemm_desc(m=m, n=n, k=k, lda=A.shape[1], ldb=B.shape[1], ldc=n, trans_a=ta, trans_b=tb,
                       prec_a=pa, prec_b=pb, prec_c=pc, math=math, cta_group=cg, max_ctas=0, alpha=alpha, beta=beta)
    wsb = ctypes.c_uint64()
    assert lib.gm_gemm_workspace_size(ctypes.byref(d), ctypes.byref(wsb)) == 0
    ws = torch.empty(max(wsb.value, 16), dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    rc = lib.gm_gemm_local(ctypes.byref(d), A.data_ptr(), B.data_ptr(), C.data_ptr(), ws.data_ptr(), wsb.value, st)
    if rc:
        return f"ERR {lib.gm_last_error().decode()}"
    torch.cuda.synchronize()
    Ad = A.double().T if ta else A.double()
    Bd = B.double().T if tb else B.double()
    ref = alpha * (Ad @ Bd) + (beta * C0.double() if beta != 0 else 0)
    err = (C.double() - ref).norm() / ref.norm()
    return float(err)

if __name__ == "__main__":
    cg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    mode = sys.argv[2] if len(sys.argv) > 2 else "check"
    if mode == "check":
        for (m, n, k) in [(128, 256, 64), (256, 256, 256), (300, 520, 260), (1024, 768, 512), (2048, 2048, 2048)]:
            for ta in (0, 1):
                for tb in (0, 1):
                    for (pa, pb, pc) in [(3, 3, 3), (0, 0, 1)]:
                        if (m * 2) % 16 and ta or (k * 2) % 16 and not ta: pass
                        e = run(m, n, k, ta, tb, pa, pb, pc, cg)
                        print(f"cg={cg} {m}x{n}x{k} ta={ta} tb={tb} prec={pa}{pb}{pc} err={e}", flush=True)
        for (pa, pb, pc, math) in [(1, 1, 1, 0), (1, 1, 1, 1), (2, 2, 2, 0), (0, 1, 1, 0), (2, 1, 0, 0)]:
            for ta, tb in [(0, 0), (1, 1), (0, 1)]:
                e = run(300, 520, 260, ta, tb, pa, pb, pc, cg, math=math)
                print(f"cg={cg} 300x520x260 ta={ta} tb={tb} prec={pa}{pb}{pc} math={math} err={e}", flush=True)
        print("beta", run(512, 512, 512, 0, 0, 3, 3, 1, cg, alpha=0.75, beta=0.5), run(512, 512, 512, 0, 0, 1, 1, 1, cg, alpha=0.75, beta=0.5))
    else:
        n = int(sys.argv[3]) if len(sys.argv) > 3 else 8192
        A = torch.randn(n, n, device="cuda", dtype=torch.bfloat16); B = torch.randn(n, n, device="cuda", dtype=torch.bfloat16)
        C = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
        import os
        caps = [int(x) for x in os.environ.get("CAPS", "0").split(",")]
        for ta, tb, cap in [(0, 0, c) for c in caps] + [(0, 1, 0), (1, 0, 0)]:
            d = L.gm_gemm_desc(m=n, n=n, k=n, lda=n, ldb=n, ldc=n, trans_a=ta, trans_b=tb, prec_a=3, prec_b=3, prec_c=3, math=0, cta_group=cg, max_ctas=cap, alpha=1.0, beta=0.0)
            st = torch.cuda.current_stream().cuda_stream
            for _ in range(3): lib.gm_gemm_local(ctypes.byref(d), A.data_ptr(), B.data_ptr(), C.data_ptr(), None, 0, st)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            it = 20
            e0.record()
            for _ in range(it): lib.gm_gemm_local(ctypes.byref(d), A.data_ptr(), B.data_ptr(), C.data_ptr(), None, 0, st)
            e1.record(); torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / it
            print(f"cg={cg} n={n} ta={ta} tb={tb} cap={cap}: {ms:.3f} ms  {2*n**3/ms/1e9:.1f} TFLOP/s", flush=True)
        for _ in range(3): torch.matmul(A, B, out=C)
        e0.record()
        for _ in range(it): torch.matmul(A, B, out=C)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / it
        print(f"torch/cuBLAS n={n}: {ms:.3f} ms  {2*n**3/ms/1e9:.1f} TFLOP/s")
