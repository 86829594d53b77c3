timeout -s KILL 900 python -m pytest tests/test_fc_gpu.py tests/test_replay_gpu.py -q -x > gpurun_out/r2an_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2an_pytest.log
tail -2 gpurun_out/r2an_pytest.log
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:line_sums -c 6 --csv python tools/dev/dev_fc_ops.py > gpurun_out/r2an_ncu.csv 2>&1
grep -E "gpu__time_duration" gpurun_out/r2an_ncu.csv | awk -F'","' '{print $NF}' | tr '\n' ' '; echo
timeout -s KILL 300 python tools/dev/dev_fc_ops.py > gpurun_out/r2an_fcops.log 2>&1; grep addRowColSum gpurun_out/r2an_fcops.log
for r in 1 2; do timeout -s KILL 300 python bench.py --config fc --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | grep '^{' | python -c "import json,sys; print('fc', json.loads(sys.stdin.read())['ms_per_step'])"; done
