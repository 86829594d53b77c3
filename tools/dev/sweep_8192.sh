for rep in 1 2 3; do
  python tools/dev/dev_cublas.py 8192 40
  python tools/dev/dev_raster.py 8192 40
done > gpurun_out/sweep8192f.txt 2>&1
python tools/dev/dev_raster.py 32768 8 >> gpurun_out/sweep8192f.txt 2>&1
timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_fc_gpu.py tests/test_hostio_gpu.py -q -x > gpurun_out/split_tests.log 2>&1
timeout 900 python -m pytest tests/test_fullsize_gpu.py -q -x -k c3 > gpurun_out/split_c3.log 2>&1
