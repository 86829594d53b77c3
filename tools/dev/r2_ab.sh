for r in 1 2; do
 for ps in 4 2 1; do
  GM_DEBUG_CONFIG=pull_streams=$ps timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 296$ps$r bench.py --gpus 4 --config fc --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | grep '^{' | python -c "import json,sys; print('N4 pull_streams=$ps', json.loads(sys.stdin.read())['ms_per_step'])"
 done
done
