# final build: 4-GPU checks and C3/FC lines at N=2/4
timeout 2700 python -m pytest tests -m gpu -q -x -rs > gpurun_out/r2hh_pytest4.log 2>&1; echo "rc=$?" >> gpurun_out/r2hh_pytest4.log
P=31500
for n in 2 4; do
P=$((P+1)); timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P bench.py --gpus $n --steps 10 --warmup 3 > gpurun_out/r2hh_bench$n.log 2>&1
P=$((P+1)); timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P bench.py --config fc --gpus $n --steps 30 --warmup 5 > gpurun_out/r2hh_fc$n.log 2>&1
done
P=$((P+1)); timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P bench.py --config fp64 --gpus 4 --steps 5 --warmup 3 > gpurun_out/r2hh_fp64_4.log 2>&1
tail -3 gpurun_out/r2hh_pytest4.log
for f in gpurun_out/r2hh_bench*.log gpurun_out/r2hh_fc*.log gpurun_out/r2hh_fp64_4.log; do echo "$f $(grep -o '"value": [0-9.]*' $f | head -3 | tr '\n' ' ') $(grep -o '"ms_per_step": [0-9.]*' $f | head -1)"; done
