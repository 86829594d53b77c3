for cfg in "tc_chunks=1" "tc_chunks=1,l2_promo=256" "tc_chunks=1,l2_promo=64" "tc_chunks=1,hint_b=1" "tc_chunks=1,hint_a=1" "tc_chunks=1,raster_group=8" "tc_chunks=1,raster_group=32" "tc_chunks=2" "tc_chunks=2,l2_promo=256"; do
echo "$cfg $(GM_DEBUG_CONFIG=$cfg timeout 120 python tools/dev/dev_one_gemm.py 8192 8192 8192 40 0)"
done
