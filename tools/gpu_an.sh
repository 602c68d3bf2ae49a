export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/an_pytest.log
timeout 300 python bench.py --workload C5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/an_c5_lt_fp64.jsonl
timeout 300 python bench.py --workload C5 --precision fp32 --no-e2e --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/an_c5_lt_fp32.jsonl
timeout 300 python bench.py --workload C5 --expo analytic --no-e2e --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/an_c5_an_fp64.jsonl
timeout 300 python bench.py --workload C5 --expo analytic --precision fp32 --no-e2e --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/an_c5_an_fp32.jsonl
cat gpurun_out/an_pytest.log
for f in gpurun_out/an_c5_*.jsonl; do python -c "import json; d=json.load(open('$f')); print('$f', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['ms_per_launch'], d['scan'])" 2>/dev/null || head -c 400 $f; done
