timeout 1800 python -m pytest tests/test_replication_gpu.py tests/test_replay_gpu.py tests/test_pipeline_gpu.py tests/test_spmd_gpu.py tests/test_checkpoint_gpu.py tests/test_hostio_gpu.py -q -x > gpurun_out/r2v_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2v_pytest.log
P=30700
for rep in 1 2; do for n in 4 2; do
P=$((P+1)); timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P bench.py --config fc --gpus $n --steps 30 --warmup 5 > gpurun_out/r2v_fc${n}_$rep.log 2>&1
done; done
P=$((P+1)); timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P tools/dev/dev_fc_spmd.py > gpurun_out/r2v_fcops4.log 2>&1
tail -2 gpurun_out/r2v_pytest.log; for f in gpurun_out/r2v_fc*_*.log; do echo "$f $(grep -o '"ms_per_step": [0-9.]*' $f)"; done; grep "step (async" gpurun_out/r2v_fcops4.log
