timeout 1800 python -m pytest tests/test_replay_gpu.py tests/test_replication_gpu.py tests/test_pipeline_gpu.py tests/test_fc_gpu.py -q -x > gpurun_out/r2j_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2j_pytest.log
timeout 300 python tools/dev/dev_fc_ops.py > gpurun_out/r2j_fcops1.log 2>&1
P=30100
for rep in 1 2; do
for cfg in "fuse_epilogue=1" "fuse_epilogue=0"; do
for n in 4 2; do
P=$((P+1)); GM_DEBUG_CONFIG=$cfg timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P bench.py --config fc --gpus $n --steps 30 --warmup 5 > gpurun_out/r2j_fc${n}_${cfg}_$rep.log 2>&1
done; done; done
timeout 300 python bench.py --config fc --steps 30 --warmup 5 > gpurun_out/r2j_fc1.log 2>&1
P=$((P+1)); timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P tools/dev/dev_fc_spmd.py > gpurun_out/r2j_fcops4.log 2>&1
for f in gpurun_out/r2j_fc*_*.log gpurun_out/r2j_fc1.log; do echo "$f $(grep -o '"ms_per_step": [0-9.]*' $f)"; done
