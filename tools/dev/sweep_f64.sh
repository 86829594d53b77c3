for rep in 1 2; do for N in 8192 16384; do python tools/dev/dev_dgemm.py $N 3; done; done > gpurun_out/f64_sweep.txt 2>&1
python -m pytest tests/test_gemm_gpu.py -q -x -k "fp64 or golden or ragged or mixed" > gpurun_out/f64_tests.log 2>&1
