set -x
nvidia-smi topo -m > gpurun_out/r2a_topo.txt 2>&1
nvidia-smi nvlink -s -i 0 > gpurun_out/r2a_nvlink_status.txt 2>&1
timeout 300 python tools/nvlink_counters.py > gpurun_out/r2a_nvml_probe.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2a_pytest.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/r2a_bench.log 2>&1
tail -3 gpurun_out/r2a_pytest.log
tail -c 1500 gpurun_out/r2a_bench.log
