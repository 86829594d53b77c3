for rep in 1 2 3; do
  python tools/dev/dev_cublas.py 8192 40
  python tools/dev/dev_raster.py 8192 40
  python tools/dev/dev_raster.py 32768 8
done > gpurun_out/sweep8192c.txt 2>&1
ncu --set full --clock-control none -k regex:tc_gemm -s 2 -c 1 -o gpurun_out/wide8192b -f python tools/dev/dev_raster.py 8192 3 > /dev/null 2>&1
python -m pytest tests/test_gemm_gpu.py -q -x > gpurun_out/stg_tests.log 2>&1
