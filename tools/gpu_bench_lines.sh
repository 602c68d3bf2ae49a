#!/bin/bash
# Bench lines of every workload on the GPU box (no tests):
#   gpurun --timeout 1500 -- 'bash tools/gpu_bench_lines.sh TAG'
# Writes gpurun_out/TAG/bench_*.jsonl and scan_stress.txt (copied to profiles/r02/TAG/ by hand after review).
set -u
TAG=${1:-bench}
O=gpurun_out/$TAG
mkdir -p "$O"
python -c "import __graft_entry__ as g; g.build()" > "$O/build.log" 2>&1 || { echo "build failed"; tail -20 "$O/build.log"; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > "$O/nvidia_smi.csv" 2>&1
B="timeout 600 python bench.py --no-cpu-baseline --no-probe"
$B > "$O/bench_c3.jsonl" 2> "$O/bench_c3.err"
$B --workload C2 --steps 20 > "$O/bench_c2.jsonl" 2> "$O/bench_c2.err"
$B --workload C5 --expo analytic --steps 10 > "$O/bench_c5an.jsonl" 2> "$O/bench_c5an.err"
$B --workload C5 --steps 10 > "$O/bench_c5lt.jsonl" 2> "$O/bench_c5lt.err"
$B --workload C4 --steps 10 > "$O/bench_c4.jsonl" 2> "$O/bench_c4.err"
$B --workload C5 --precision fp32 --steps 10 > "$O/bench_c5lt_fp32.jsonl" 2> "$O/bench_c5lt_fp32.err"
$B --workload C5 --expo analytic --precision fp32 --steps 10 > "$O/bench_c5an_fp32.jsonl" 2> "$O/bench_c5an_fp32.err"
$B --workload G1 > "$O/bench_g1.jsonl" 2> "$O/bench_g1.err"
for n in 2 4 8; do
  $B --emulate-ranks $n --no-e2e > "$O/bench_c3_rankof$n.jsonl" 2> "$O/bench_c3_rankof$n.err" || true
  $B --workload C4 --steps 10 --emulate-ranks $n --no-e2e > "$O/bench_c4_rankof$n.jsonl" 2> "$O/bench_c4_rankof$n.err" || true
done
timeout 300 python tools/c2_dt_sweep.py > "$O/c2_dt_sweep.txt" 2>&1
timeout 300 python tools/scan_stress.py > "$O/scan_stress.txt" 2>&1
for f in "$O"/bench_*.jsonl; do
  python - "$f" <<'EOF'
import json, sys
for l in open(sys.argv[1]):
    try:
        d = json.loads(l)
    except ValueError:
        continue
    r = d.get("roofline", {}); s = d.get("scan", {}) or {}; e = d.get("e2e") or {}
    print(sys.argv[1].split("/")[-1], f"{d['value']:.4g}", f"ms/step {d['ms_per_step']:.4g}", f"frac {r.get('frac', 0):.3f}",
          f"int_ms {r.get('ms_per_launch', 0):.4g}", f"scan_ms {s.get('ms_per_launch', 0) or 0:.4g}",
          f"e2e {e.get('value', 0) or 0:.4g}", f"pred {(d.get('emulated') or {}).get('predicted_value', 0):.4g}")
EOF
done
cat "$O/scan_stress.txt" "$O/c2_dt_sweep.txt"
