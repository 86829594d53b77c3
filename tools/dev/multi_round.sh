TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29513"
timeout 300 $TR --nproc-per-node 4 tools/dev/h2d_probe.py > gpurun_out/h2d_n4.txt 2>&1
timeout 600 $TR --nproc-per-node 2 bench.py --gpus 2 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err
timeout 600 $TR --nproc-per-node 4 bench.py --gpus 4 --config fp64 > gpurun_out/bench_fp64_n4.json 2> gpurun_out/bench_fp64_n4.err
timeout 600 $TR --nproc-per-node 4 bench.py --gpus 4 --config fc > gpurun_out/bench_fc_n4.json 2> gpurun_out/bench_fc_n4.err
timeout 900 $TR --nproc-per-node 4 tools/spmd_check.py > gpurun_out/spmd_check_n4.txt 2>&1
