timeout 2400 python -m pytest tests -m gpu -q -x -rs > gpurun_out/r2u_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2u_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2u_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2u_smoke.log
timeout 600 python bench.py > gpurun_out/r2u_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2u_bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2u_launches.csv \
    python bench.py --steps 2 --warmup 3 --e2e-steps 1 --dependent-steps 0 --no-cpu-baseline --no-c2 > gpurun_out/r2u_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 3 -c 1 -o gpurun_out/r2u_prof_bench -f \
    python bench.py --steps 2 --warmup 3 --e2e-steps 0 --dependent-steps 0 --no-cpu-baseline --no-c2 > gpurun_out/r2u_ncu_full.log 2>&1
timeout 300 python bench.py --config fc --steps 30 --warmup 5 > gpurun_out/r2u_fc1.log 2>&1
timeout 300 python bench.py --config fp64 --steps 5 --warmup 3 > gpurun_out/r2u_fp64.log 2>&1
tail -3 gpurun_out/r2u_pytest.log
