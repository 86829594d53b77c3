timeout 1200 python -m pytest tests/test_gemm_gpu.py tests/test_fc_gpu.py tests/test_replay_gpu.py tests/test_device_gpu.py tests/test_fullsize_gpu.py tests/test_pipeline_gpu.py -q -x > gpurun_out/r2n_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2n_pytest.log
timeout 600 python tools/dev/dev_c2_sweep.py > gpurun_out/r2n_c2.log 2>&1
timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2n_bench1.log 2>&1
timeout 300 python bench.py --config fc --steps 30 --warmup 5 > gpurun_out/r2n_fc1.log 2>&1
tail -3 gpurun_out/r2n_pytest.log; cat gpurun_out/r2n_c2.log; grep -o '"value": [0-9.]*' gpurun_out/r2n_bench1.log | head -2; grep -o '"ms_per_step": [0-9.]*' gpurun_out/r2n_fc1.log
