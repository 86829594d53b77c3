timeout 1500 python -m pytest tests/test_spmd_gpu.py -q -x -k headline > gpurun_out/r2q_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2q_pytest.log
P=30500; P=$((P+1)); timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P tools/spmd_fullsize.py > gpurun_out/r2q_full4.log 2>&1
tail -3 gpurun_out/r2q_pytest.log; grep SPMD_FULLSIZE gpurun_out/r2q_full4.log
