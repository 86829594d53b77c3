TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29591"
timeout 600 $TR --nproc-per-node 4 tools/dev/dev_fc_spmd.py > gpurun_out/fc_spmd_n4b.txt 2>&1
