GM_DEBUG_CONFIG=panel_min_gflop=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 30601 tools/spmd_check.py > gpurun_out/r2r_spmd8.log 2>&1; echo "rc=$?" >> gpurun_out/r2r_spmd8.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 30602 tools/spmd_fullsize.py > gpurun_out/r2r_full8.log 2>&1; echo "rc=$?" >> gpurun_out/r2r_full8.log
grep -h "SPMD_\|rank0" gpurun_out/r2r_spmd8.log gpurun_out/r2r_full8.log
