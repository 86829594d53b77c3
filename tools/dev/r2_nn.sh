for r in 1 2 3; do
 for gr in 1 0; do
  GM_DEBUG_CONFIG=graph_replay=$gr timeout -s KILL 200 python bench.py --config fc --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r2nn_fc_g${gr}_$r.log 2>&1
 done
done
timeout -s KILL 900 python -m pytest tests/test_replay_gpu.py tests/test_fc_gpu.py tests/test_spmd_gpu.py tests/test_pipeline_gpu.py -q -x > gpurun_out/r2nn_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2nn_pytest.log
tail -3 gpurun_out/r2nn_pytest.log
for f in gpurun_out/r2nn_fc_g*; do echo $f; python - "$f" <<'PY'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(d.get('ms_per_step'), d.get('value'), d.get('host_issue_ms_per_step'))
    elif 'Error' in l: print(l[:300])
PY
done
