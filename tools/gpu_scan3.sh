# scan3 A/B: default (hints, 16 stages) vs variants; parity first
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -k "scan or spin" -x -q 2>&1 | tail -3
for lib in libspinsim_b200.so; do
  export SPINSIM_LIB=$PWD/paper_2204_05586_b200/$lib
  timeout 300 python tools/scan_stress.py | grep scan
  for wl in C5; do timeout 300 python bench.py --workload $wl --steps 5 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$lib', '$wl', d['value'], d['ms_per_step'], d.get('scan'))"; done
done
unset SPINSIM_LIB
timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan3 -c 1 -f -o gpurun_out/prof_scan3_stress python tools/scan_stress.py 2>&1 | tail -1
