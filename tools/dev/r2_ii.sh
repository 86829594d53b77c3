timeout 1500 python -m pytest tests/test_gemm_gpu.py tests/test_fc_gpu.py tests/test_replay_gpu.py tests/test_device_gpu.py tests/test_fullsize_gpu.py tests/test_pipeline_gpu.py -q -x > gpurun_out/r2ii_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2ii_pytest.log
timeout 600 python tools/dev/dev_c2_sweep.py > gpurun_out/r2ii_c2.log 2>&1
timeout 300 python bench.py --config fc --steps 30 --warmup 5 > gpurun_out/r2ii_fc1.log 2>&1
timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2ii_bench1.log 2>&1
tail -2 gpurun_out/r2ii_pytest.log; cat gpurun_out/r2ii_c2.log; grep -o '"ms_per_step": [0-9.]*' gpurun_out/r2ii_fc1.log; grep -o '"value": [0-9.]*\|"config2_bf16_8192_tflops": [0-9.]*\|"sm_mhz": [0-9.]*' gpurun_out/r2ii_bench1.log | head -4
