# round-2 check: GPU tests (2 GPUs), NVML probe, bench N=1/2, FC N=1/2
timeout 300 python tools/nvlink_counters.py > gpurun_out/r2b_nvml_probe.log 2>&1
timeout 900 python -m pytest tests/test_pipeline_gpu.py -x -q > gpurun_out/r2b_pipe.log 2>&1
echo "pipe rc=$?" >> gpurun_out/r2b_pipe.log
timeout 1800 python -m pytest tests -m gpu -q -x --deselect tests/test_pipeline_gpu.py > gpurun_out/r2b_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2b_pytest.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2b_bench1.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/r2b_bench2.log 2>&1
timeout 300 python bench.py --config fc --steps 20 --warmup 5 > gpurun_out/r2b_fc1.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --config fc --gpus 2 --steps 20 --warmup 5 > gpurun_out/r2b_fc2.log 2>&1
tail -3 gpurun_out/r2b_pipe.log gpurun_out/r2b_pytest.log
tail -c 600 gpurun_out/r2b_bench2.log
