# NVML 2 ms clock sampling inside short timed regions (C2, C4) + the default line
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/s10_clocks; mkdir -p $O
timeout 300 python bench.py --workload C2 2>&1 | tail -1 > $O/bench_c2.jsonl
timeout 300 python bench.py --workload C4 2>&1 | tail -1 > $O/bench_c4.jsonl
timeout 600 python bench.py --no-cpu-baseline 2>&1 | tail -1 > $O/bench_default.jsonl
python -c "
import json
for f in ['c2','c4','default']:
    d=json.load(open('$O/bench_'+f+'.jsonl')); print(f, d['value'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])
"
