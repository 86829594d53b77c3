timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_fc_gpu.py tests/test_replay_gpu.py -q -x > gpurun_out/r2p_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2p_pytest.log
P=30300
for rep in 1 2; do for n in 4 2; do
P=$((P+1)); timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P bench.py --config fc --gpus $n --steps 30 --warmup 5 > gpurun_out/r2p_fc${n}_$rep.log 2>&1
done; done
timeout 300 python bench.py --config fc --steps 30 --warmup 5 > gpurun_out/r2p_fc1.log 2>&1
P=$((P+1)); timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $P tools/dev/dev_fc_spmd.py > gpurun_out/r2p_fcops4.log 2>&1
tail -2 gpurun_out/r2p_pytest.log; for f in gpurun_out/r2p_fc*.log; do echo "$f $(grep -o '"ms_per_step": [0-9.]*' $f)"; done
