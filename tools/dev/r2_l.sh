timeout 600 python tools/dev/dev_c2_sweep.py > gpurun_out/r2l_c2.log 2>&1
GM_DEBUG_CONFIG=tc_chunks=1 timeout 600 python tools/dev/dev_c2_sweep.py > gpurun_out/r2l_c2_narrow.log 2>&1
GM_DEBUG_CONFIG=tc_sync=0 timeout 600 python tools/dev/dev_c2_sweep.py > gpurun_out/r2l_c2_nosync.log 2>&1
cat gpurun_out/r2l_c2*.log
./tools/dev/memop_probe > gpurun_out/r2l_memop.log 2>&1
cat gpurun_out/r2l_memop.log
