GM_DEBUG_CONFIG=sm_copy=1 timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611 tools/spmd_check.py > gpurun_out/r2ac_spmd4.log 2>&1; echo "spmd rc=$?"; grep -E "SPMD_CHECK|False" gpurun_out/r2ac_spmd4.log | head -5
for r in 1 2; do
 for sc in 1 0; do
  for n in 4 2; do
  GM_DEBUG_CONFIG=sm_copy=$sc timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 297$n$sc$r bench.py --gpus $n --config fc --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N$n sm_copy=$sc', d['ms_per_step'], d['bytes_received_per_step']['max_rank'])"
  done
 done
done
GM_DEBUG_CONFIG=sm_copy=1 timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29622 bench.py --gpus 4 --no-c2 --no-cpu-baseline > gpurun_out/r2ac_c3_4.log 2>&1
python -c "
import json
for l in open('gpurun_out/r2ac_c3_4.log'):
    if l.startswith('{'):
        d=json.loads(l); print('C3 N4 sm_copy=1', d['value'], 'dep', d.get('dependent',{}).get('value'), 'exch', d.get('nvlink',{}).get('exchange_ms'), 'clk', d.get('clocks',{}).get('sm_mhz'))"
