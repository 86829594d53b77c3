for cfg in "pdl=0" "tc_sync=0" "tc_chunks=1" "fuse_epilogue=0" "tma_store=0" "pdl=0,tc_sync=0"; do
  echo "== $cfg" >> gpurun_out/r2mm.log
  GM_DEBUG_CONFIG=$cfg timeout -s KILL 120 python bench.py --config fc --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | grep -E "GmError|ms_per_step" | cut -c1-300 >> gpurun_out/r2mm.log
done
cat gpurun_out/r2mm.log
