for cfg in "verbose=0" "flag_barrier=0" "panel_k=4096,a_chunk_rows=8192,b_chunk_cols=4096"; do
echo "== $cfg" >> gpurun_out/r2e_ab.log
GM_DEBUG_CONFIG=$cfg timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 tools/dev/dev_pipe_ab.py 2>&1 | grep -v "OMP\|^\*\|NCCL" >> gpurun_out/r2e_ab.log
done
