timeout -s KILL 3000 python -m pytest tests -m gpu -q -x > gpurun_out/r2uu_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2uu_pytest.log
for n in 2 4; do
  timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2957$n bench.py --gpus $n > gpurun_out/r2uu_bench$n.log 2>&1
  timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2958$n bench.py --gpus $n --config fc --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r2uu_fc$n.log 2>&1
done
tail -3 gpurun_out/r2uu_pytest.log
for f in gpurun_out/r2uu_bench*.log gpurun_out/r2uu_fc*.log; do echo $f; grep '^{' $f | cut -c1-300; done
