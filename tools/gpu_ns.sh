export PATH=/usr/local/cuda/bin:$PATH
for v in "" ns2 ns3; do
  lib=$PWD/paper_2204_05586_b200/libspinsim_b200${v:+.$v}.so
  echo "== ${v:-ns5}"
  SPINSIM_LIB=$lib timeout 300 python bench.py --workload C5 --expo analytic --no-e2e --no-cpu-baseline --no-probe 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C5an', d['value'], d['ms_per_step'], d['scan'])"
  SPINSIM_LIB=$lib timeout 300 python bench.py --workload C2 --no-e2e --no-cpu-baseline --no-probe 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C2', d['value'], d['ms_per_step'], d['scan'])"
  SPINSIM_LIB=$lib timeout 300 python tools/scan_stress.py 2>&1 | tail -3
done
SPINSIM_LIB=$PWD/paper_2204_05586_b200/libspinsim_b200.ns2.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -2
SPINSIM_LIB=$PWD/paper_2204_05586_b200/libspinsim_b200.ns3.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -2
