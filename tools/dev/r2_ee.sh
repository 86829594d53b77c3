timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_pipeline_gpu.py tests/test_fc_gpu.py tests/test_replay_gpu.py -q -x > gpurun_out/r2ee_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2ee_pytest.log
for rep in 1 2; do for cfg in pdl=1 pdl=0; do
GM_DEBUG_CONFIG=$cfg timeout 600 python tools/dev/dev_c2_sweep.py > gpurun_out/r2ee_c2_${cfg}_$rep.log 2>&1
GM_DEBUG_CONFIG=$cfg timeout 300 python bench.py --config fc --steps 30 --warmup 5 > gpurun_out/r2ee_fc_${cfg}_$rep.log 2>&1
echo "$cfg $rep"; grep "ours" gpurun_out/r2ee_c2_${cfg}_$rep.log; grep -o '"ms_per_step": [0-9.]*' gpurun_out/r2ee_fc_${cfg}_$rep.log
done; done
tail -2 gpurun_out/r2ee_pytest.log
