# round-1 closing check: every GPU test and smoke on the final HEAD
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/s10_close; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3 > $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 600 python bench.py 2>&1 | tail -1 > $O/bench_default.jsonl
cat $O/pytest_gpu.log $O/smoke.log; head -c 400 $O/bench_default.jsonl
