timeout -s KILL 600 python -m pytest tests/test_fc_gpu.py tests/test_replay_gpu.py tests/test_pipeline_gpu.py -q -x > gpurun_out/r2ww_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2ww_pytest.log
tail -2 gpurun_out/r2ww_pytest.log
for m in 0 2; do
  GM_DEBUG_CONFIG=ls_mode=$m timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:line_sums -c 6 --csv python tools/dev/dev_fc_ops.py > gpurun_out/r2ww_ncu_m$m.csv 2>&1
  echo "mode $m"; grep -E "gpu__time_duration" gpurun_out/r2ww_ncu_m$m.csv | awk -F'","' '{print $NF}' | tr '\n' ' '; echo
done
timeout -s KILL 300 python bench.py --config fc --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r2ww_fc.log 2>&1
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:line_sums -c 2 -o gpurun_out/r2ww_prof_ls -f python tools/dev/dev_fc_ops.py > /dev/null 2>&1
grep '^{' gpurun_out/r2ww_fc.log | cut -c1-100; python -c "
import json
for l in open('gpurun_out/r2ww_fc.log'):
    if l.startswith('{'): print(json.loads(l)['ms_per_step'])"
