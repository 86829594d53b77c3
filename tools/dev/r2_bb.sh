timeout 900 python -m pytest tests/test_gemm_gpu.py -q -x -k "fold or tf32 or config2 or layout" > gpurun_out/r2bb_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2bb_pytest.log
timeout 600 python - > gpurun_out/r2bb_fold.log 2>&1 <<'PY'
import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "oracle"))
import numpy as np, oracle as O
from paper_1611_07819_b200 import gridmath as G
n = 8192
for math in (0, 2):
    with G.Session(workers=1) as s:
        one = G.makeSingleTileLayout(n, n, 0)
        A = s.createMatrix(n, n, G.Precision.BF16, one); B = s.createMatrix(n, n, G.Precision.BF16, one)
        C = s.createMatrix(n, n, G.Precision.Single, one)
        s.fillUniform(A, 1); s.fillUniform(B, 2)
        for _ in range(3): G.gemm(s, A, B, C, 1.0, 0.0, math=math)
        s.timerStart()
        for _ in range(10): s.gemmAsync(A, B, C) if math == 0 else G.gemm(s, A, B, C, 1.0, 0.0, math=math)
        ms = s.timerStop() / 10
        c = s.getDataRaw(C); a = s.getDataRaw(A); b = s.getDataRaw(B)
    rows = (1000, 1016)
    want = O.gemm_c(n, n, n, a, 3, b, 3, np.zeros((n, n), np.float32), 1, 1.0, 0.0, 0, 0, rows)
    print(f"math={math} 8192^3 bf16->f32 {ms:.3f} ms {2*n**3/ms/1e9:.1f} TFLOP/s rel_fro vs reference chain {O.rel_fro(c[rows[0]:rows[1]], want[rows[0]:rows[1]]):.3e}")
PY
tail -3 gpurun_out/r2bb_pytest.log; cat gpurun_out/r2bb_fold.log
