# wave-aligned two-chunk host pipeline (C2 e2e): new parity test, host-API tests, C2 bench line with e2e
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out/s10
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "host_api" 2>&1 | tail -3 > gpurun_out/s10/pytest_pair.log
for i in 1 2; do timeout 300 python bench.py --workload C2 --no-cpu-baseline 2>&1 | tail -1 >> gpurun_out/s10/bench_c2_pair.jsonl; done
timeout 300 python bench.py --workload C2 --no-cpu-baseline --chunks 1 2>&1 | tail -1 >> gpurun_out/s10/bench_c2_pair.jsonl
cat gpurun_out/s10/pytest_pair.log
python -c "
import json
for l in open('gpurun_out/s10/bench_c2_pair.jsonl'):
    d=json.loads(l); print(d['value'], d['ms_per_step'], d['e2e'])
"
