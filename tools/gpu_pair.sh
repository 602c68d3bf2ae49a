export PATH=/usr/local/cuda/bin:$PATH
for v in "" pair4 pair3; do
  lib=$PWD/paper_2204_05586_b200/libspinsim_b200${v:+.$v}.so
  SPINSIM_LIB=$lib timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-probe 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${v:-base}', 'C3', d['value'], d['roofline']['frac'], d['roofline']['ms_per_launch'], d['clocks']['sm_mhz'])"
done
SPINSIM_LIB=$PWD/paper_2204_05586_b200/libspinsim_b200.pair3.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
