# scan3 parity + ncu captures (scan-stress spin-half, C5 spin-one)
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -k "scan or spin" -x -q 2>&1 | tail -3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan3 -c 1 -f -o gpurun_out/prof_scan3_stress python tools/scan_stress.py 2>&1 | tail -3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan3 -s 3 -c 1 -f -o gpurun_out/prof_scan3_c5 python bench.py --workload C5 --steps 3 --warmup 3 2>&1 | tail -3
