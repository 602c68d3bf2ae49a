# Interval-kernel change check: the full GPU suite, smoke, the bench lines of the 3×3 paths (C3 default, C2, C5
# Lie–Trotter FP64, G1) and the executed-flop table.   gpurun -- 'bash tools/gpu_kernel_check.sh TAG'
set -u
O=gpurun_out/${1:-kcheck}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
B="timeout 600 python bench.py --no-cpu-baseline --no-probe"
$B > $O/bench_c3.jsonl 2>/dev/null
$B --workload C2 --steps 20 > $O/bench_c2.jsonl 2>/dev/null
$B --workload C5 --steps 10 > $O/bench_c5lt.jsonl 2>/dev/null
$B --workload G1 > $O/bench_g1.jsonl 2>/dev/null
tail -3 $O/pytest_gpu.log; tail -2 $O/smoke.log
for f in $O/*.jsonl; do echo $f; python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d.get('roofline') or {}; e=d.get('e2e') or {}
print(d['value'], d['ms_per_step'], r.get('frac'), r.get('ms_per_launch'), e.get('value'), (d.get('paper_benchmark') or {}).get('roofline_frac'))"; done
