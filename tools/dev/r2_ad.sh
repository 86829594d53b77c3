GM_DEBUG_CONFIG=sm_copy=1,verbose=1 CUDA_LAUNCH_BLOCKING=1 timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29631 tools/spmd_check.py > gpurun_out/r2ad_spmd2.log 2>&1; echo "rc=$?"
grep -E "SPMD|sm copy|GmError|illegal" gpurun_out/r2ad_spmd2.log | head -30
