timeout -s KILL 3000 python -m pytest tests -m gpu -q -x > gpurun_out/r2ah_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2ah_pytest.log
tail -3 gpurun_out/r2ah_pytest.log
