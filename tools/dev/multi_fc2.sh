TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29517"
./tools/dev/ce2d_probe > gpurun_out/ce2d.txt 2>&1
timeout 600 $TR --nproc-per-node 4 tools/dev/dev_fc_spmd.py > gpurun_out/fc_spmd_n4.txt 2>&1
