# final-build multi-GPU record: full GPU suite on 4 GPUs, C3 bench N=2/4 (dependent + e2e), pipelining A/B N=4, fp64 N=4
timeout 2700 python -m pytest tests -m gpu -q -x -rs > gpurun_out/r2w_pytest4.log 2>&1; echo "rc=$?" >> gpurun_out/r2w_pytest4.log
P=30900
for n in 2 4; do
P=$((P+1)); timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P bench.py --gpus $n --steps 10 --warmup 3 > gpurun_out/r2w_bench$n.log 2>&1
done
P=$((P+1)); timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P tools/dev/dev_pipe_ab.py > gpurun_out/r2w_ab4.log 2>&1
P=$((P+1)); timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P bench.py --config fp64 --gpus 4 --steps 5 --warmup 3 > gpurun_out/r2w_fp64_4.log 2>&1
tail -3 gpurun_out/r2w_pytest4.log; grep -h "C3\|FC" gpurun_out/r2w_ab4.log
for f in gpurun_out/r2w_bench*.log gpurun_out/r2w_fp64_4.log; do echo "$f $(grep -o '"value": [0-9.]*' $f | head -3 | tr '\n' ' ')"; done
