# after factoring the host-pipeline plan out (ss_host_chunk_plan): all GPU tests, C2/C4/C3 lines with e2e
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/s10_plan; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3 > $O/pytest_gpu.log
timeout 300 python bench.py --workload C2 --no-cpu-baseline 2>&1 | tail -1 > $O/bench_c2.jsonl
timeout 300 python bench.py --workload C4 --no-cpu-baseline 2>&1 | tail -1 > $O/bench_c4.jsonl
timeout 600 python bench.py 2>&1 | tail -1 > $O/bench_default.jsonl
cat $O/pytest_gpu.log
python -c "
import json
for f in ['c2','c4','default']:
    d=json.load(open('$O/bench_'+f+'.jsonl')); print(f, d['value'], d['e2e']['value'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['samples'])
"
