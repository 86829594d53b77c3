timeout -s KILL 600 python -m pytest tests/test_replay_gpu.py -q -x 2>&1 | tail -1
p=29800
for r in 1 2; do
 for gr in 1 0; do
  for n in 1 4; do
  p=$((p+1))
  GM_DEBUG_CONFIG=graph_replay=$gr timeout -s KILL 150 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $p bench.py --gpus $n --config fc --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r2ai_fc_n${n}_g${gr}_$r.log 2>&1
  grep '^{' gpurun_out/r2ai_fc_n${n}_g${gr}_$r.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N$n graph=$gr', d['ms_per_step'], d['host_issue_ms_per_step'])"
  done
 done
done
