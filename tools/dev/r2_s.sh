# lockstep / raster sweep at 32768^3: DRAM bytes + time per launch (ncu, one launch each), then bench for 3 configs
for cfg in "tc_sync=16,raster_group=16" "tc_sync=8,raster_group=16" "tc_sync=4,raster_group=16" "tc_sync=32,raster_group=16" "tc_sync=8,raster_group=12" "tc_sync=16,raster_group=12" "tc_sync=8,raster_group=8"; do
GM_DEBUG_CONFIG=$cfg timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:tc_gemm -s 1 -c 1 --csv python tools/dev/dev_one_gemm.py 32768 32768 32768 2 > "gpurun_out/r2s_$cfg.csv" 2>&1
echo "$cfg"; grep -E "dram__bytes|gpu__time|cycles_elapsed|tensor" "gpurun_out/r2s_$cfg.csv" | awk -F'","' '{print "   ", $(NF-2), $(NF)}'
done
