# FC step breakdown at N=2 with / without panel flags; C3 N=2 bench
for PF in 1 0; do
GM_DEBUG_CONFIG=panel_flags=$PF timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2952$PF tools/dev/dev_fc_spmd.py > gpurun_out/r2c_fcops_pf$PF.log 2>&1
GM_DEBUG_CONFIG=panel_flags=$PF timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2953$PF bench.py --gpus 2 --steps 10 --warmup 3 --e2e-steps 0 > gpurun_out/r2c_bench2_pf$PF.log 2>&1
done
nvidia-smi nvlink -gt d -i 0 > gpurun_out/r2c_nvlink_gt.txt 2>&1
nvidia-smi nvlink -gt d -i 0 >> gpurun_out/r2c_nvlink_gt.txt 2>&1
ls /usr/bin | grep -i dcgm > gpurun_out/r2c_dcgm.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c_smoke_ncu.log 2>&1
echo "smoke ncu rc=$?" >> gpurun_out/r2c_smoke_ncu.log
