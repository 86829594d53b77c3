# one GPU: line-sums parity + timing, N=1 bench, ncu launch list + full capture of the top kernel, FC N=1 + launch list
timeout 900 python -m pytest tests/test_fc_gpu.py tests/test_replay_gpu.py -q -x > gpurun_out/r2h_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2h_pytest.log
timeout 300 python tools/dev/dev_fc_ops.py > gpurun_out/r2h_fcops1.log 2>&1
timeout 400 python bench.py --steps 10 --warmup 3 > gpurun_out/r2h_bench1.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2h_launches.csv \
    python bench.py --steps 2 --warmup 3 --e2e-steps 1 --dependent-steps 0 --no-cpu-baseline --no-c2 > gpurun_out/r2h_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 3 -c 1 -o gpurun_out/r2h_prof_bench -f \
    python bench.py --steps 2 --warmup 3 --e2e-steps 0 --dependent-steps 0 --no-cpu-baseline --no-c2 > gpurun_out/r2h_ncu_full.log 2>&1
timeout 300 python bench.py --config fc --steps 20 --warmup 5 > gpurun_out/r2h_fc1.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2h_fc_launches.csv \
    python bench.py --config fc --steps 3 --warmup 3 > gpurun_out/r2h_ncu_fc.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:line_sums -c 2 -o gpurun_out/r2h_prof_ls -f \
    python tools/dev/dev_fc_ops.py > gpurun_out/r2h_ncu_ls.log 2>&1
