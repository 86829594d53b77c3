timeout 900 python -m pytest tests/test_pipeline_gpu.py -q -x > gpurun_out/r2y_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2y_pytest.log
P=31100
P=$((P+1)); timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P tools/dev/dev_pipe_ab.py > gpurun_out/r2y_ab4.log 2>&1
P=$((P+1)); timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $P tools/dev/dev_pipe_ab.py > gpurun_out/r2y_ab2.log 2>&1
P=$((P+1)); timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 4 --steps 10 --warmup 3 --e2e-steps 0 > gpurun_out/r2y_bench4.log 2>&1
tail -2 gpurun_out/r2y_pytest.log; grep -h "C3" gpurun_out/r2y_ab4.log gpurun_out/r2y_ab2.log; grep -o '"value": [0-9.]*' gpurun_out/r2y_bench4.log
