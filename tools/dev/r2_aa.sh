P=31300
P=$((P+1)); AB_ROUNDS=7 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P tools/dev/dev_pipe_ab.py > gpurun_out/r2aa_ab4.log 2>&1
P=$((P+1)); AB_ROUNDS=7 GM_DEBUG_CONFIG=lockstep_data=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P tools/dev/dev_pipe_ab.py > gpurun_out/r2aa_ab4_nold.log 2>&1
grep -h C3 gpurun_out/r2aa_ab4.log gpurun_out/r2aa_ab4_nold.log
