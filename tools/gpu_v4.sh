export PATH=/usr/local/cuda/bin:$PATH
export SPINSIM_LIB=$PWD/paper_2204_05586_b200/libspinsim_b200.v5.so
timeout 600 python -m pytest tests -m gpu -q -x -k "scan or c5 or c2 or spin or partition or large or rand" 2>&1 | tail -3
for v in v5 ""; do
  export SPINSIM_LIB=$PWD/paper_2204_05586_b200/libspinsim_b200${v:+.$v}.so
  echo "== ${v:-v3}"
  timeout 300 python bench.py --workload C5 --expo analytic --no-e2e --no-cpu-baseline --no-probe 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C5an', d['value'], d['ms_per_step'], d['scan'])"
  timeout 300 python bench.py --workload C5 --no-e2e --no-cpu-baseline --no-probe 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C5lt', d['value'], d['ms_per_step'], d['scan']['achieved'])"
  timeout 300 python tools/scan_stress.py 2>&1 | tail -3
done
