timeout -s KILL 600 python -m pytest tests/test_fc_gpu.py tests/test_replay_gpu.py -q -x > gpurun_out/r2ss_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2ss_pytest.log
timeout -s KILL 300 python tools/dev/dev_fc_ops.py > gpurun_out/r2ss_fcops1.log 2>&1
timeout -s KILL 300 python tools/dev/dev_fc_ops.py > gpurun_out/r2ss_fcops2.log 2>&1
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:line_sums -c 2 -o gpurun_out/r2ss_prof_ls -f python tools/dev/dev_fc_ops.py > gpurun_out/r2ss_ncu_ls.log 2>&1
tail -2 gpurun_out/r2ss_pytest.log; head -1 gpurun_out/r2ss_fcops1.log; head -1 gpurun_out/r2ss_fcops2.log
