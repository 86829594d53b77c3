for rg in 8 12 16 24 32; do
  GM_DEBUG_CONFIG=raster_group=$rg timeout -s KILL 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:tc_gemm -c 1 --csv python tools/dev/dev_one_gemm.py 32768 32768 32768 1 > gpurun_out/r2af_rg$rg.csv 2>&1
  echo "rg=$rg $(grep -E 'dram__bytes|gpu__time' gpurun_out/r2af_rg$rg.csv | awk -F'","' '{print $(NF-2)"="$NF}' | tr '\n' ' ')"
done
for rg in 8 16 32; do
  GM_DEBUG_CONFIG=raster_group=$rg timeout -s KILL 300 python tools/dev/dev_one_gemm.py 32768 32768 32768 12 2>&1 | tail -1 | sed "s/^/rg=$rg timed: /"
done
