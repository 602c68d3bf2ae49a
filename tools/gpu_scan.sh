# Scan-kernel change check: every scan parity test, the scan paths table, the bench lines whose states pass changed.
#   gpurun -- 'bash tools/gpu_scan.sh TAG'
set -u
O=gpurun_out/${1:-scan}
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "scan or chain or parity or compact or fused" > $O/pytest_scan.log 2>&1; echo "rc=$?" >> $O/pytest_scan.log
timeout 600 python tools/scan_paths.py > $O/scan_paths.txt 2>&1
B="timeout 600 python bench.py --no-cpu-baseline --no-probe --no-secondary"
for n in 2 4 8; do $B --emulate-ranks $n --no-e2e > $O/bench_c3_rankof$n.jsonl 2>/dev/null; done
$B --workload G1 --emulate-ranks 8 --no-e2e > $O/bench_g1_rankof8.jsonl 2>/dev/null
$B --workload C5 --steps 10 > $O/bench_c5lt.jsonl 2>/dev/null
tail -3 $O/pytest_scan.log; cat $O/scan_paths.txt
for f in $O/*.jsonl; do echo $f; python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d.get('roofline') or {}; s=d.get('scan') or {}; em=d.get('emulated') or {}
print(d['value'], d['ms_per_step'], r.get('frac'), s.get('ms_per_launch'), s.get('frac'), em.get('predicted_value'))"; done
