for cfg in "tc_chunks=2" "tc_chunks=1"; do
GM_DEBUG_CONFIG=$cfg timeout 600 ncu --set full --clock-control none -k regex:tc_gemm -s 2 -c 1 -o gpurun_out/r2m_$cfg -f python tools/dev/dev_one_gemm.py 8192 8192 4096 3 > gpurun_out/r2m_$cfg.log 2>&1
done
timeout 600 ncu --set full --clock-control none -k regex:nvjet -s 2 -c 1 -o gpurun_out/r2m_cublas -f python tools/dev/dev_cublas.py 8192 3 > gpurun_out/r2m_cublas.log 2>&1
ls -la gpurun_out/r2m*
