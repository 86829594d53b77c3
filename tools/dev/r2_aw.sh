timeout -s KILL 1500 python -m pytest tests/test_spmd_gpu.py tests/test_replay_gpu.py -q -x -k "not headline" > gpurun_out/r2aw_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2aw_pytest.log; tail -2 gpurun_out/r2aw_pytest.log
p=30050
for r in 1 2; do
 for z in 1 0; do
  for n in 4 2; do
  p=$((p+1))
  GM_DEBUG_CONFIG=fuse_zero_sums=$z timeout -s KILL 150 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $p bench.py --gpus $n --config fc --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r2aw_fc_n${n}_z${z}_$r.log 2>&1
  grep '^{' gpurun_out/r2aw_fc_n${n}_z${z}_$r.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N$n zero_sums=$z', d['ms_per_step'])"
  done
 done
done
