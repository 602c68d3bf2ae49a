export PATH=/usr/local/cuda/bin:$PATH
export SPINSIM_LIB=$PWD/paper_2204_05586_b200/libspinsim_b200.v6.so
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "scan" 2>&1 | tail -3
timeout 300 python -m pytest tests -m gpu -q -x -k "c5 or large or long or rand or spin" 2>&1 | tail -2
for v in v6 ""; do
  export SPINSIM_LIB=$PWD/paper_2204_05586_b200/libspinsim_b200${v:+.$v}.so
  echo "== ${v:-v3}"
  timeout 120 python bench.py --workload C5 --expo analytic --no-e2e --no-cpu-baseline --no-probe 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C5an', d['value'], d['ms_per_step'], d['scan']['achieved'], d['scan']['ms_per_launch'])"
  timeout 120 python tools/scan_stress.py 2>&1 | tail -3
done
