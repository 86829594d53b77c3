GM_DEBUG_CONFIG=tc_chunks=2 timeout 600 python tools/dev/dev_c2_sweep.py > gpurun_out/r2o_c2_wide.log 2>&1
timeout 600 python tools/dev/dev_c2_sweep.py > gpurun_out/r2o_c2.log 2>&1
cat gpurun_out/r2o_c2_wide.log gpurun_out/r2o_c2.log
