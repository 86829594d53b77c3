# 4-GPU round-2 evidence: SPMD parity (4 ranks NCCL/IPC; 8 ranks = 2x4 grid on 4 GPUs via gloo control),
# pipelining A/B at N=4, C3 bench N=2/4 (+dependent), FC step N=2/4
timeout 1800 python -m pytest tests/test_spmd_gpu.py tests/test_pipeline_gpu.py tests/test_dropin_cpp.py -q -x -rs > gpurun_out/r2f_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2f_pytest.log
P=29700
for n in 4 2; do
P=$((P+1)); timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P bench.py --gpus $n --steps 10 --warmup 3 > gpurun_out/r2f_bench$n.log 2>&1
P=$((P+1)); timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P bench.py --config fc --gpus $n --steps 20 --warmup 5 > gpurun_out/r2f_fc$n.log 2>&1
done
P=$((P+1)); timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P tools/dev/dev_pipe_ab.py > gpurun_out/r2f_ab4.log 2>&1
P=$((P+1)); timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P tools/dev/dev_fc_spmd.py > gpurun_out/r2f_fcops4.log 2>&1
tail -3 gpurun_out/r2f_pytest.log
