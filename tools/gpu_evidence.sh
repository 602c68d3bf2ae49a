#!/bin/bash
# Round-2 evidence run on the GPU box:  gpurun --timeout 3000 -- 'bash tools/gpu_evidence.sh TAG [tests|bench|profile|all]'
# Writes gpurun_out/TAG/ (copied to profiles/r02/TAG/ by hand after review):
#   tests:   pytest -m gpu, smoke()
#   bench:   the default bench line (C3 + the paper's benchmark), the reference arm
#   profile: the ncu launch list of the default bench command (per-launch times, --clock-control none), one
#            `ncu --set full` capture of the C3 interval kernel and of the fused run chain (summaries), the executed-flop
#            table (tools/executed_flops.py), the SASS excerpt (tools/sass_excerpt.py)
set -u
TAG=${1:-r02}
WHAT=${2:-all}
O=gpurun_out/$TAG
mkdir -p "$O"
python -c "import __graft_entry__ as g; g.build()" > "$O/build.log" 2>&1 || { echo "build failed"; tail -20 "$O/build.log"; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > "$O/nvidia_smi.csv" 2>&1
nproc > "$O/host_cores.txt"
if [ "$WHAT" = "tests" ] || [ "$WHAT" = "all" ]; then
  timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -rf --durations=15 > "$O/pytest_gpu.log" 2>&1
  echo "pytest rc=$?" >> "$O/pytest_gpu.log"
  timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > "$O/smoke.log" 2>&1
fi
if [ "$WHAT" = "bench" ] || [ "$WHAT" = "all" ]; then
  timeout 900 python bench.py > "$O/bench_default.jsonl" 2> "$O/bench_default.err"
  timeout 900 python bench.py --impl reference > "$O/bench_reference.jsonl" 2> "$O/bench_reference.err"
fi
if [ "$WHAT" = "profile" ] || [ "$WHAT" = "all" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$O/launches_default.csv" \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-probe --no-e2e --no-secondary > /dev/null 2>&1
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:interval_kernel -s 1 -c 1 \
    -o "$O/c3_interval" python tools/profile_run.py --workload C3 --batch 1024 > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:run_chain -s 1 -c 1 \
    -o "$O/run_chain" python tools/profile_run.py --workload C4S --evaluate > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none -k regex:chain_kernel -s 1 -c 1 \
    -o "$O/chain" python tools/profile_run.py --workload C3 --evaluate > /dev/null 2>&1
  for r in c3_interval run_chain chain; do python tools/ncu_summary.py "$O/$r.ncu-rep" > "$O/ncu_$r.txt" 2>&1; done
  timeout 1200 python tools/executed_flops.py "$O" > "$O/flops.log" 2>&1
  python tools/sass_excerpt.py > "$O/sass_excerpt.txt" 2>&1
fi
tail -5 "$O"/pytest_gpu.log 2>/dev/null
head -c 400 "$O"/bench_default.jsonl 2>/dev/null
