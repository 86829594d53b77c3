# the driver's round-end checks on a 1-GPU box: full GPU suite + smoke + default bench
timeout 2400 python -m pytest tests -m gpu -q -x -rs > gpurun_out/r2k_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2k_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2k_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2k_smoke.log
timeout 600 python bench.py > gpurun_out/r2k_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2k_bench.log
timeout 600 python bench.py --impl reference > gpurun_out/r2k_ref.log 2>&1; echo "rc=$?" >> gpurun_out/r2k_ref.log
tail -3 gpurun_out/r2k_pytest.log
