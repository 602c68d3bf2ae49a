# run-to-run spread of the default bench line (C3) and of C2 at the default 5 steps and at 20 steps
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/s10_rep; mkdir -p $O
for i in 1 2 3; do
  timeout 600 python bench.py --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3', d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" >> $O/repeat.txt
done
for st in 5 20 50; do
  timeout 300 python bench.py --workload C2 --no-cpu-baseline --no-e2e --no-probe --steps $st 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C2 steps=$st', d['value'], d['ms_per_step'], d['roofline']['frac'])" >> $O/repeat.txt
done
cat $O/repeat.txt
