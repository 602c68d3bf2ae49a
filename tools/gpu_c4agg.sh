export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/agg_pytest.log
timeout 300 python bench.py --workload C4 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/agg_bench_c4.jsonl
timeout 300 python bench.py --workload C4 --gpus 2 --share-gpu --dist-backend gloo --no-e2e --no-cpu-baseline 2>&1 | tail -1 > /dev/null
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --workload C4 --gpus 2 --share-gpu --dist-backend gloo --no-cpu-baseline --steps 3 2>&1 | tail -1 > gpurun_out/agg_bench_c4_2rank_shared.jsonl
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/agg_launches_c4.csv python bench.py --workload C4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-probe > /dev/null 2>&1
cat gpurun_out/agg_pytest.log
python -c "import json; d=json.load(open('gpurun_out/agg_bench_c4.jsonl')); print(d['value'], d['ms_per_step'], d['exchange_and_scan_ms'], d['roofline']['frac'], d.get('e2e'))"
head -c 600 gpurun_out/agg_bench_c4_2rank_shared.jsonl; echo
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/agg_launches_c4.csv')) if len(r)>10]
hdr=rows[0]; ki=hdr.index('Kernel Name'); vi=hdr.index('Metric Value')
for r in rows[1:][-8:]: print(r[ki][:60], r[vi])
PY
