TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
rm -f gpurun_out/repl_ring2.txt
for rep in 1 2; do
  timeout 300 $TR --master-port 2953$rep --nproc-per-node 4 tools/dev/dev_repl.py 2>&1 | grep "N=" >> gpurun_out/repl_ring2.txt
  timeout 600 $TR --master-port 2954$rep --nproc-per-node 4 bench.py --gpus 4 --config fc 2>/dev/null | grep '^{' >> gpurun_out/repl_ring2.txt
done
timeout 600 $TR --master-port 29560 --nproc-per-node 2 bench.py --gpus 2 --config fc 2>/dev/null | grep '^{' >> gpurun_out/repl_ring2.txt
timeout 900 $TR --master-port 29550 --nproc-per-node 4 tools/spmd_check.py > gpurun_out/spmd_check_ring2.txt 2>&1
