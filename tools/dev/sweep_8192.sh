for rep in 1 2 3; do
  python tools/dev/dev_cublas.py 8192 40
  python tools/dev/dev_raster.py 8192 40
done > gpurun_out/sweep8192g.txt 2>&1
python tools/dev/dev_raster.py 32768 8 >> gpurun_out/sweep8192g.txt 2>&1
