for r in 1 2; do
 for gr in 1 0; do
  GM_DEBUG_CONFIG=graph_replay=$gr timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2954$r bench.py --gpus 4 --config fc --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r2oo_fc4_g${gr}_$r.log 2>&1
  GM_DEBUG_CONFIG=graph_replay=$gr timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2955$r bench.py --gpus 2 --config fc --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r2oo_fc2_g${gr}_$r.log 2>&1
 done
done
for f in gpurun_out/r2oo_fc*; do echo $f; python - "$f" <<'PY'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(d.get('ms_per_step'), d.get('value'), d.get('host_issue_ms_per_step'), d.get('bytes_received_per_step'))
    elif 'Error' in l: print(l[:300])
PY
done
