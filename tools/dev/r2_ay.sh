timeout -s KILL 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2ay_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2ay_pytest.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2ay_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2ay_smoke.log
timeout -s KILL 900 python bench.py > gpurun_out/r2ay_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2ay_bench.log
timeout -s KILL 600 python bench.py --impl reference > gpurun_out/r2ay_bench_ref.log 2>&1
tail -3 gpurun_out/r2ay_pytest.log; tail -2 gpurun_out/r2ay_smoke.log; tail -2 gpurun_out/r2ay_bench.log | cut -c1-600
