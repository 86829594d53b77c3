timeout -s KILL 1500 python -m pytest tests/test_spmd_gpu.py tests/test_replay_gpu.py -q -x -k "not headline" > gpurun_out/r2pp_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2pp_pytest.log
GM_DEBUG_CONFIG=graph_replay=1 timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29561 tools/spmd_check.py > gpurun_out/r2pp_spmd4_nccl_graph.log 2>&1; echo "rc=$?" >> gpurun_out/r2pp_spmd4_nccl_graph.log
tail -3 gpurun_out/r2pp_pytest.log; grep -E "FC step|SPMD_CHECK|rc=" gpurun_out/r2pp_spmd4_nccl_graph.log
