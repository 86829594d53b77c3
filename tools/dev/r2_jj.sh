timeout 900 python -m pytest tests/test_fc_gpu.py tests/test_replay_gpu.py -q -x > gpurun_out/r2jj_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2jj_pytest.log
timeout 300 python tools/dev/dev_fc_ops.py > gpurun_out/r2jj_fcops1.log 2>&1
timeout 300 ncu --set full --clock-control none -k regex:line_sums -c 2 -o gpurun_out/r2jj_prof_ls -f python tools/dev/dev_fc_ops.py > gpurun_out/r2jj_ncu_ls.log 2>&1
tail -2 gpurun_out/r2jj_pytest.log; head -2 gpurun_out/r2jj_fcops1.log
