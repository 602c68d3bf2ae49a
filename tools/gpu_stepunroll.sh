export PATH=/usr/local/cuda/bin:$PATH
for v in "" su2 su4; do
  lib=$PWD/paper_2204_05586_b200/libspinsim_b200${v:+.$v}.so
  for w in C4; do
  SPINSIM_LIB=$lib timeout 300 python bench.py --workload $w --no-e2e --no-cpu-baseline --no-probe 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${v:-su1}', '$w', d['value'], d['roofline']['ms_per_launch'])"
  done
  SPINSIM_LIB=$lib timeout 300 python bench.py --workload C5 --expo analytic --no-e2e --no-cpu-baseline --no-probe 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${v:-su1}', 'C5an', d['value'], d['roofline']['ms_per_launch'])"
  SPINSIM_LIB=$lib timeout 300 python bench.py --workload C2 --no-e2e --no-cpu-baseline --no-probe 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${v:-su1}', 'C2', d['value'], d['roofline']['ms_per_launch'])"
done
