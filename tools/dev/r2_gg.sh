# final build: 1-GPU driver-style checks
timeout 2400 python -m pytest tests -m gpu -q -x -rs > gpurun_out/r2gg_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2gg_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2gg_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2gg_smoke.log
timeout 600 python bench.py > gpurun_out/r2gg_bench.log 2>&1; echo "rc=$?" >> gpurun_out/r2gg_bench.log
timeout 600 python bench.py --impl reference > gpurun_out/r2gg_ref.log 2>&1
timeout 300 python bench.py --config fc --steps 30 --warmup 5 > gpurun_out/r2gg_fc1.log 2>&1
tail -3 gpurun_out/r2gg_pytest.log; tail -1 gpurun_out/r2gg_smoke.log
python3 -c "
import json
d=[json.loads(l) for l in open('gpurun_out/r2gg_bench.log') if l.startswith('{')][0]
print(d['value'], d['roofline']['frac'], d['roofline']['frac_clock_normalised'], d['clocks']['sm_mhz'], d['e2e']['value'], d.get('config2_bf16_8192_tflops'), d['gpu_launches'])"
