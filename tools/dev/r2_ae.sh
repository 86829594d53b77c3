p=29700
for r in 1 2; do
 for sc in 1 0; do
  for n in 4 2; do
  p=$((p+1))
  GM_DEBUG_CONFIG=sm_copy=$sc timeout -s KILL 150 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $p bench.py --gpus $n --config fc --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r2ae_fc_n${n}_s${sc}_$r.log 2>&1
  grep '^{' gpurun_out/r2ae_fc_n${n}_s${sc}_$r.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N$n sm_copy=$sc', d['ms_per_step'], d['bytes_received_per_step']['max_rank'])"
  done
 done
done
