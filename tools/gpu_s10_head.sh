# session-4 restart check on the rebuilt HEAD: all GPU tests, smoke, default bench line, C2 line
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out/s10
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/s10/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s10/smoke.log 2>&1
timeout 600 python bench.py 2>&1 | tail -1 > gpurun_out/s10/bench_default.jsonl
timeout 300 python bench.py --workload C2 2>&1 | tail -1 > gpurun_out/s10/bench_c2.jsonl
cat gpurun_out/s10/pytest_gpu.log gpurun_out/s10/smoke.log
for f in gpurun_out/s10/bench_*.jsonl; do echo "$f: $(head -c 300 $f)"; done
