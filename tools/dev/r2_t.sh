# sustained A/B of the lockstep period at 32768^3 (bench N=1, alternating) + K sweep with tc_sync=8
for rep in 1 2; do for cfg in "tc_sync=16" "tc_sync=8"; do
GM_DEBUG_CONFIG=$cfg timeout 300 python bench.py --steps 20 --warmup 3 --e2e-steps 0 --dependent-steps 0 --no-cpu-baseline --no-c2 > "gpurun_out/r2t_${cfg}_${rep}.log" 2>&1
echo "$cfg $rep $(grep -o '"value": [0-9.]*' "gpurun_out/r2t_${cfg}_${rep}.log" | head -1) $(grep -o '"sm_mhz": [0-9.]*' "gpurun_out/r2t_${cfg}_${rep}.log")"
done; done
GM_DEBUG_CONFIG=tc_sync=8 timeout 600 python tools/dev/dev_c2_sweep.py > gpurun_out/r2t_c2_sync8.log 2>&1
timeout 600 python tools/dev/dev_c2_sweep.py > gpurun_out/r2t_c2_sync16.log 2>&1
cat gpurun_out/r2t_c2_sync8.log gpurun_out/r2t_c2_sync16.log
