# Profiles for the current build (one GPU): bench launch list, one full
# capture of the bench's GEMM launch, DRAM bytes of the per-GPU ops at N=2/4/8.
set -x
python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-c2 > gpurun_out/prof_bench_plain.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-c2 > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 3 -c 1 -o gpurun_out/prof_bench -f \
    python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-c2 > gpurun_out/ncu_full.log 2>&1
for N in 2 4 8; do
  python tools/dev/traffic_shapes.py $N 3 > gpurun_out/shape_time_$N.txt 2>&1
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
      --clock-control none -k regex:tc_gemm -s 2 -c 2 --csv python tools/dev/traffic_shapes.py $N 2 > gpurun_out/shape_ncu_$N.csv 2>&1
done
