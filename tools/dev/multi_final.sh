TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $TR --master-port 29581 --nproc-per-node 4 tools/spmd_check.py > gpurun_out/spmd_check_final4.txt 2>&1
timeout 900 $TR --master-port 29582 --nproc-per-node 2 tools/spmd_check.py > gpurun_out/spmd_check_final2.txt 2>&1
python -m pytest tests/test_spmd_gpu.py -q > gpurun_out/spmd_gpu_final.log 2>&1
timeout 600 $TR --master-port 29583 --nproc-per-node 4 bench.py --gpus 4 > gpurun_out/bench_final4.json 2> gpurun_out/bench_final4.err
timeout 600 $TR --master-port 29584 --nproc-per-node 2 bench.py --gpus 2 > gpurun_out/bench_final2.json 2> gpurun_out/bench_final2.err
timeout 600 $TR --master-port 29585 --nproc-per-node 4 bench.py --gpus 4 --config fc > gpurun_out/bench_final_fc4.json 2>&1
timeout 600 $TR --master-port 29586 --nproc-per-node 4 bench.py --gpus 4 --impl reference > gpurun_out/bench_final_ref4.json 2>&1
