# line sums TMA path parity + timing; pipelining A/B at N=4/2 with the local/remote stream split; sanitizers
timeout 900 python -m pytest tests/test_fc_gpu.py -q -x > gpurun_out/r2g_fc_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_fc_pytest.log
CUDA_VISIBLE_DEVICES=0 timeout 300 python tools/dev/dev_fc_ops.py > gpurun_out/r2g_fcops1.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29801 tools/dev/dev_pipe_ab.py > gpurun_out/r2g_ab4.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29802 tools/dev/dev_pipe_ab.py > gpurun_out/r2g_ab2.log 2>&1
for t in memcheck racecheck synccheck; do
CUDA_VISIBLE_DEVICES=0 timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_driver.py > gpurun_out/r2g_san_$t.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_san_$t.log
done
