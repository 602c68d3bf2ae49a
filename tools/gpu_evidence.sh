#!/bin/bash
# Round-2 evidence run on the GPU box:  gpurun --timeout 2400 -- 'bash tools/gpu_evidence.sh TAG [tests|bench|all]'
# Writes gpurun_out/TAG/ (copied to profiles/r02/TAG/ by hand after review).
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
fi
tail -5 "$O"/pytest_gpu.log 2>/dev/null
cat "$O"/bench_default.jsonl 2>/dev/null | head -c 600
