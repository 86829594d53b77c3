python tools/dev/dev_die.py > gpurun_out/die_map.txt 2>&1
for rep in 1 2 3; do for D in 0 1; do GM_DIE_AWARE=$D timeout 120 python tools/dev/dev_raster.py 32768 16; done; done > gpurun_out/die_time.txt 2>&1
for D in 0 1; do GM_DIE_AWARE=$D timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,lts__t_sectors_srcunit_ltcfabric.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:tc_gemm -s 2 -c 1 --csv python tools/dev/dev_raster.py 32768 3 > gpurun_out/die_ncu_$D.csv 2>&1; done
