TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29519"
timeout 300 $TR --nproc-per-node 4 tools/dev/dev_repl.py > gpurun_out/repl_n4.txt 2>&1
timeout 300 $TR --nproc-per-node 2 tools/dev/dev_repl.py > gpurun_out/repl_n2.txt 2>&1
