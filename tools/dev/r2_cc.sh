timeout 1200 python -m pytest tests/test_gemm_gpu.py tests/test_fc_gpu.py tests/test_replay_gpu.py tests/test_device_gpu.py tests/test_pipeline_gpu.py -q -x > gpurun_out/r2cc_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2cc_pytest.log
GM_DEBUG_CONFIG=tc_chunks=1 timeout 600 python tools/dev/dev_c2_sweep.py > gpurun_out/r2cc_c2_narrow.log 2>&1
timeout 600 python tools/dev/dev_c2_sweep.py > gpurun_out/r2cc_c2.log 2>&1
timeout 600 python - > gpurun_out/r2cc_fold.log 2>&1 <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
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
        for _ in range(10): G.gemm(s, A, B, C, 1.0, 0.0, math=math)
        ms = s.timerStop() / 10
    print(f"math={math} 8192^3 bf16->f32 {ms:.3f} ms {2*n**3/ms/1e9:.1f} TFLOP/s")
PY
timeout 300 python bench.py --config fc --steps 30 --warmup 5 > gpurun_out/r2cc_fc1.log 2>&1
tail -2 gpurun_out/r2cc_pytest.log; cat gpurun_out/r2cc_c2_narrow.log gpurun_out/r2cc_c2.log gpurun_out/r2cc_fold.log; grep -o '"ms_per_step": [0-9.]*' gpurun_out/r2cc_fc1.log
