for n in 1 2 4; do
timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2959$n tools/dev/dev_fc_timeline.py > gpurun_out/r2ak_tl$n.log 2>&1
tail -6 gpurun_out/r2ak_tl$n.log
done
