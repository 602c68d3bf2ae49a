export PATH=/usr/local/cuda/bin:$PATH
for v in "" u1 u4 u8; do
  lib=$PWD/paper_2204_05586_b200/libspinsim_b200${v:+.$v}.so
  SPINSIM_LIB=$lib timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-probe 2>&1 | tail -1 > gpurun_out/un_c3_${v:-u2}.jsonl
  SPINSIM_LIB=$lib timeout 300 python bench.py --workload G1 --no-e2e --no-cpu-baseline --no-probe 2>&1 | tail -1 > gpurun_out/un_g1_${v:-u2}.jsonl
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/un_launches_c4.csv python bench.py --workload C4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-probe > /dev/null 2>&1
for f in gpurun_out/un_*.jsonl; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d['value'], d['roofline']['frac'], d['roofline']['ms_per_launch'], d['clocks']['sm_mhz'])" 2>/dev/null || head -c 300 $f; done
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/un_launches_c4.csv')) if len(r)>10]
hdr=rows[0]; ki=hdr.index('Kernel Name'); vi=hdr.index('Metric Value')
for r in rows[1:][-12:]: print(r[ki][:60], r[vi])
PY
