for tb in 0 1; do for cfg in tc_chunks=1 tc_chunks=2; do
GM_DEBUG_CONFIG=$cfg timeout 120 python tools/dev/dev_one_gemm.py 8192 8192 8192 40 $tb
done; done
