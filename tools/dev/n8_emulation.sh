# 8 ranks on a 4-GPU box (2 per GPU): does NCCL accept it, and does the 2x4
# grid's SPMD path (IPC plane incl. same-device peers) pass spmd_check?
nvidia-smi topo -m > gpurun_out/topo4.txt 2>&1
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29511"
timeout 180 $TR --nproc-per-node 8 tools/dev/nccl_dup_probe.py > gpurun_out/n8_nccl_probe.txt 2>&1
if ! grep -q FAIL gpurun_out/n8_nccl_probe.txt && grep -q "ok" gpurun_out/n8_nccl_probe.txt; then
  timeout 1200 $TR --nproc-per-node 8 tools/spmd_check.py > gpurun_out/n8_spmd_check.txt 2>&1
  echo "spmd_check exit $?" >> gpurun_out/n8_spmd_check.txt
fi
timeout 600 $TR --nproc-per-node 4 bench.py --gpus 4 > gpurun_out/bench_n4.json 2> gpurun_out/bench_n4.err
