TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $TR --master-port 29521 --nproc-per-node 4 tools/spmd_check.py > gpurun_out/spmd_check_n4b.txt 2>&1
timeout 900 $TR --master-port 29522 --nproc-per-node 2 tools/spmd_check.py > gpurun_out/spmd_check_n2b.txt 2>&1
python -m pytest tests/test_spmd_gpu.py -q > gpurun_out/spmd_gpu_test.log 2>&1
timeout 600 $TR --master-port 29523 --nproc-per-node 4 bench.py --gpus 4 > gpurun_out/bench_n4c.json 2> gpurun_out/bench_n4c.err
timeout 600 $TR --master-port 29524 --nproc-per-node 2 bench.py --gpus 2 > gpurun_out/bench_n2c.json 2> gpurun_out/bench_n2c.err
