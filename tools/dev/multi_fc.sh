TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29515"
timeout 600 $TR --nproc-per-node 4 bench.py --gpus 4 --config fc > gpurun_out/bench_fc_n4b.json 2> gpurun_out/bench_fc_n4b.err
timeout 600 $TR --nproc-per-node 2 bench.py --gpus 2 --config fc > gpurun_out/bench_fc_n2b.json 2> gpurun_out/bench_fc_n2b.err
python bench.py --config fc > gpurun_out/bench_fc_n1d.json 2>&1
python -m pytest tests/test_gemm_gpu.py -q -x -k "wide or invariance or golden" > gpurun_out/wide_tests.log 2>&1
