# A/B of GEMM kernel builds (variants/lib_<commit>.so swapped in place).
cp paper_1611_07819_b200/libgridmath_b200.so /tmp/lib_keep.so
for rep in 1 2; do
for V in bb9b727 5100ebe ee2c29d 251e323 HEAD; do
  cp variants/lib_$V.so paper_1611_07819_b200/libgridmath_b200.so
  echo "== $V rep $rep" >> gpurun_out/ab.txt
  python tools/dev/traffic_shapes.py 2 3 >> gpurun_out/ab.txt 2>&1
  python tools/dev/dev_raster.py 32768 6 2>&1 | cut -c1-90 >> gpurun_out/ab.txt
  if [ $rep = 1 ]; then
    ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:tc_gemm -s 2 -c 1 --csv python tools/dev/traffic_shapes.py 2 2 2>&1 | grep -E '"(dram|gpu__|sm__)' | awk -F'","' '{print $(NF-2), $NF}' >> gpurun_out/ab.txt
  fi
done
done
cp /tmp/lib_keep.so paper_1611_07819_b200/libgridmath_b200.so
