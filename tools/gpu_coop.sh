export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for v in ""; do
  export SPINSIM_LIB=$PWD/paper_2204_05586_b200/libspinsim_b200${v:+.$v}.so
  for w in C2 C4; do
    timeout 300 python bench.py --workload $w --no-e2e --no-cpu-baseline --no-probe 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${v:-cps128}', '$w', d['value'], d['ms_per_step'], d.get('scan', {}).get('ms_per_launch'), d.get('exchange_and_scan_ms'))"
  done
done
