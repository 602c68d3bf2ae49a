# final HEAD check of session 4: all GPU tests, smoke, default bench line
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/s10_end; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3 > $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 600 python bench.py 2>&1 | tail -1 > $O/bench_default.jsonl
timeout 300 python bench.py --workload C4 --no-cpu-baseline 2>&1 | tail -1 > $O/bench_c4.jsonl
timeout 300 python bench.py --workload C2 --no-cpu-baseline 2>&1 | tail -1 > $O/bench_c2.jsonl
cat $O/pytest_gpu.log $O/smoke.log
python -c "
import json
for f in ['default','c4','c2']:
    d=json.load(open('$O/bench_'+f+'.jsonl')); print(f, d['value'], d['e2e']['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['samples'], d['gpu_launches'])
"
