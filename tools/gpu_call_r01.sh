export PATH=/usr/local/cuda/bin:$PATH
timeout 600 python bench.py 2>&1 | tail -1 > gpurun_out/r01_bench_default.jsonl
timeout 300 python bench.py --workload C4 --steps 3 2>&1 | tail -1 > gpurun_out/r01_bench_c4.jsonl
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 2 --no-e2e --no-cpu-baseline --no-probe 2>&1 | tail -1 > gpurun_out/r01_bench_torchrun1.jsonl
timeout 300 python bench.py --workload C5 --steps 3 --no-e2e --no-cpu-baseline --no-probe 2>&1 | tail -1 > gpurun_out/r01_bench_c5_fp64.jsonl
timeout 300 python bench.py --workload C5 --precision fp32 --steps 3 --no-e2e --no-cpu-baseline --no-probe 2>&1 | tail -1 > gpurun_out/r01_bench_c5_fp32.jsonl
timeout 300 python bench.py --workload C2 --steps 3 --no-e2e --no-cpu-baseline --no-probe 2>&1 | tail -1 > gpurun_out/r01_bench_c2.jsonl
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 2>&1 | tail -1 > gpurun_out/r01_bench_reference.jsonl
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-probe > /dev/null 2>&1
nproc > gpurun_out/host_info.txt; lscpu | grep -E "Model name|Socket|Thread|Core" >> gpurun_out/host_info.txt; nvidia-smi >> gpurun_out/host_info.txt
for f in gpurun_out/r01_bench_*.jsonl; do echo "$f: $(head -c 300 $f)"; done
