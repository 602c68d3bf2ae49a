# Chain-kernel ring experiment (round 2, s33/s34): scan parity tests, every scan kernel on the paper-shaped problems,
# the C3 per-rank shard lines and the default C3 line.   gpurun -- 'bash tools/gpu_s33.sh TAG'
set -u
O=gpurun_out/${1:-s34_chain}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/nvidia_smi.csv 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "scan or chain or parity" > $O/pytest_scan.log 2>&1; echo "rc=$?" >> $O/pytest_scan.log
timeout 600 python tools/scan_paths.py > $O/scan_paths.txt 2>&1
for n in 2 4 8; do timeout 600 python bench.py --emulate-ranks $n --no-cpu-baseline --no-e2e --no-secondary --no-probe > $O/bench_c3_rankof$n.jsonl 2>$O/err_$n.txt; done
timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-secondary --no-probe > $O/bench_c3.jsonl 2>$O/err_c3.txt
tail -3 $O/pytest_scan.log
cat $O/scan_paths.txt
for f in $O/*.jsonl; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d.get('roofline',{}).get('frac'), d.get('scan',{}).get('ms_per_launch'), d.get('scan',{}).get('frac'))"; done
