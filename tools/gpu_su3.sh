# general spin-one (su(3)) path: parity tests, full GPU suite (regression), G1 bench for the occupancy variants, C3
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_gpu_su3.py -q -x 2>&1 | tail -15 > gpurun_out/su3_pytest.log
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/su3_pytest_all.log
for v in "" mb3 mb2; do
  lib=paper_2204_05586_b200/libspinsim_b200${v:+.$v}.so
  SPINSIM_LIB=$PWD/$lib timeout 300 python bench.py --workload G1 --no-e2e --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/su3_bench_g1_${v:-mb4}.jsonl
done
timeout 300 python bench.py --workload G1 --precision fp32 --no-e2e --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/su3_bench_g1_fp32.jsonl
timeout 600 python bench.py --no-e2e --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/su3_bench_c3.jsonl
cat gpurun_out/su3_pytest.log gpurun_out/su3_pytest_all.log
for f in gpurun_out/su3_bench_*.jsonl; do echo "$f: $(head -c 300 $f)"; python -c "import json,sys; d=json.load(open('$f')); print(d['value'], d['roofline']['frac'], d['roofline']['ms_per_launch'])" 2>/dev/null; done
