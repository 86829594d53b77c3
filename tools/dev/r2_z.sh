P=31200
for cfg in "lockstep_data=0,tc_sync=8" "lockstep_data=1,tc_sync=8" "lockstep_data=1,tc_sync=16" "lockstep_data=1,tc_sync=16,class_sort=0" "lockstep_data=0,tc_sync=16,class_sort=0"; do
P=$((P+1)); GM_DEBUG_CONFIG=$cfg timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $P tools/dev/dev_pipe_ab.py > "gpurun_out/r2z_$cfg.log" 2>&1
echo "== $cfg"; grep C3 "gpurun_out/r2z_$cfg.log"
done
