timeout -s KILL 240 python bench.py --config fc --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2ll_fc_g1.log 2>&1
GM_DEBUG_CONFIG=panel_min_gflop=0 timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29533 tools/spmd_check.py > gpurun_out/r2ll_spmd2.log 2>&1; echo "rc=$?" >> gpurun_out/r2ll_spmd2.log
timeout -s KILL 600 python -m pytest tests/test_replay_gpu.py -q -x > gpurun_out/r2ll_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2ll_pytest.log
nvidia-smi --query-compute-apps=pid,name --format=csv >> gpurun_out/r2ll_pytest.log
tail -3 gpurun_out/r2ll_fc_g1.log | cut -c1-400; tail -4 gpurun_out/r2ll_spmd2.log; tail -3 gpurun_out/r2ll_pytest.log
