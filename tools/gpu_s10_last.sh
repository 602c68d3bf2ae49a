# session-4 last evidence set (after the staged cooperative scan): all GPU tests, smoke, every bench line, reference arm, torchrun N=1, launch list,
# FP64 op counters and ncu --set full captures of the top kernels (summarised by tools/ncu_summary.py)
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/s10_last; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3 > $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 600 python bench.py 2>&1 | tail -1 > $O/bench_default.jsonl
timeout 300 python bench.py --workload C2 2>&1 | tail -1 > $O/bench_c2.jsonl
timeout 300 python bench.py --workload C4 2>&1 | tail -1 > $O/bench_c4.jsonl
timeout 300 python bench.py --workload C5 --expo lie_trotter --no-cpu-baseline 2>&1 | tail -1 > $O/bench_c5_lt_fp64.jsonl
timeout 300 python bench.py --workload C5 --expo lie_trotter --precision fp32 --no-e2e --no-cpu-baseline 2>&1 | tail -1 > $O/bench_c5_lt_fp32.jsonl
timeout 300 python bench.py --workload C5 --expo analytic --no-e2e --no-cpu-baseline 2>&1 | tail -1 > $O/bench_c5_an_fp64.jsonl
timeout 300 python bench.py --workload G1 --no-cpu-baseline 2>&1 | tail -1 > $O/bench_g1.jsonl
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 1 --steps 3 --no-cpu-baseline 2>&1 | tail -1 > $O/bench_torchrun1.jsonl
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 2>&1 | tail -1 > $O/bench_reference.jsonl
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-probe > /dev/null 2>&1
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__inst_executed.sum,gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active
timeout 300 ncu --metrics $M --clock-control none -k regex:interval_kernel -s 1 -c 1 --csv python tools/profile_run.py --workload C3 --batch 1024 > $O/flops_c3.csv 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:interval_kernel -s 1 -c 1 -o gpurun_out/s10l_interval_c3 python tools/profile_run.py --workload C3 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:chain_kernel -s 1 -c 1 -o gpurun_out/s10l_chain_c3 python tools/profile_run.py --workload C3 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:interval_kernel -s 1 -c 1 -o gpurun_out/s10l_interval_c2 python tools/profile_run.py --workload C2 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/s10l_interval_c3.ncu-rep gpurun_out/s10l_chain_c3.ncu-rep gpurun_out/s10l_interval_c2.ncu-rep > $O/ncu_summary.txt 2>&1
cat $O/pytest_gpu.log $O/smoke.log
for f in $O/bench_*.jsonl; do echo "$f: $(head -c 200 $f)"; done
