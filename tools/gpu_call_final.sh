# end-of-milestone check: all GPU tests, smoke, the default bench line, C4/C2/C5 lines, torchrun path, launch list
export PATH=/usr/local/cuda/bin:$PATH
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/final_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1
timeout 600 python bench.py 2>&1 | tail -1 > gpurun_out/final_bench_default.jsonl
timeout 300 python bench.py --workload C4 2>&1 | tail -1 > gpurun_out/final_bench_c4.jsonl
timeout 300 python bench.py --workload C2 --no-e2e --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/final_bench_c2.jsonl
timeout 300 python bench.py --workload C5 --precision fp32 --no-e2e --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/final_bench_c5_fp32.jsonl
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 1 --steps 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/final_bench_torchrun1.jsonl
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 2>&1 | tail -1 > gpurun_out/final_bench_reference.jsonl
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-probe > /dev/null 2>&1
cat gpurun_out/final_pytest_gpu.log gpurun_out/final_smoke.log
for f in gpurun_out/final_bench_*.jsonl; do echo "$f: $(head -c 250 $f)"; done
