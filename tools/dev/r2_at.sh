p=30020
for r in 1 2; do
for cfg in "lazy_written=1,war_side=1" "lazy_written=0,war_side=0"; do
  p=$((p+1))
  GM_DEBUG_CONFIG=$cfg AB_ROUNDS=5 timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $p tools/dev/dev_pipe_ab.py > gpurun_out/r2at_ab4_$p.log 2>&1
  echo "== cfg='$cfg'"; grep "C3" gpurun_out/r2at_ab4_$p.log | cut -c1-85
done
done
