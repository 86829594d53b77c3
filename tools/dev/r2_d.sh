# panel-pipelining experiment matrix at N=2 (C3 bench: independent, dependent, isolated exchange)
run() { tag=$1; cfg=$2; GM_DEBUG_CONFIG=$cfg timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $3 bench.py --gpus 2 --steps 10 --warmup 3 --e2e-steps 0 > gpurun_out/r2d_$tag.log 2>&1; }
run pf0 panel_flags=0 29601
run pf1 panel_flags=1 29602
run pk4096 panel_k=4096,a_chunk_rows=8192,b_chunk_cols=4096 29603
run pk8192 panel_k=8192,a_chunk_rows=8192,b_chunk_cols=4096 29604
run pf1nosync tc_sync=0 29605
run pf0nosync panel_flags=0,tc_sync=0 29606
GM_DEBUG_CONFIG=panel_flags=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29607 tools/dev/dev_fc_spmd.py > gpurun_out/r2d_fcops_pf1.log 2>&1
for f in gpurun_out/r2d_*.log; do echo $f; python3 -c "
import json,sys
for l in open('$f'):
    if l.startswith('{'):
        d=json.loads(l); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms_per_gemm'], 'dep', d['dependent']['value'], d['dependent']['ms_per_step'], 'xchg', d['nvlink']['exchange_ms'], d['clocks']['sm_mhz'])
"; done
