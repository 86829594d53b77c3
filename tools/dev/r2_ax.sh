timeout -s KILL 3000 python -m pytest tests -m gpu -q -x > gpurun_out/r2ax_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2ax_pytest.log
tail -3 gpurun_out/r2ax_pytest.log
for n in 2 4; do
  timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2960$n bench.py --gpus $n > gpurun_out/r2ax_bench$n.log 2>&1
  timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2961$n bench.py --gpus $n --config fc --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r2ax_fc$n.log 2>&1
done
for f in gpurun_out/r2ax_bench2.log gpurun_out/r2ax_bench4.log gpurun_out/r2ax_fc2.log gpurun_out/r2ax_fc4.log; do python -c "
import json,sys
for l in open('$f'):
    if l.startswith('{'):
        d=json.loads(l); print('$f', d['value'], d['ms_per_step'], (d.get('dependent') or {}).get('value'), (d.get('e2e') or {}).get('value'), (d.get('clocks') or {}).get('sm_mhz'))"; done
