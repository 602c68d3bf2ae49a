export PATH=/usr/local/cuda/bin:$PATH
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > gpurun_out/ty_pytest_all.log
timeout 600 python bench.py --no-e2e --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/ty_bench_c3.jsonl
timeout 300 python bench.py --workload G1 --no-e2e --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/ty_bench_g1.jsonl
timeout 300 python bench.py --workload C2 --no-e2e --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/ty_bench_c2.jsonl
timeout 300 python bench.py --workload C5 --precision fp32 --no-e2e --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/ty_bench_c5_fp32.jsonl
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__inst_executed.sum,gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active
timeout 300 ncu --metrics $M --clock-control none -k regex:interval_kernel -s 1 -c 1 --csv python tools/profile_run.py --workload C3 --batch 1024 > gpurun_out/ty_flops_c3.csv 2>&1
timeout 300 ncu --metrics $M --clock-control none -k regex:interval_kernel -s 1 -c 1 --csv python tools/profile_run.py --workload G1 --batch 1024 > gpurun_out/ty_flops_g1.csv 2>&1
cat gpurun_out/ty_pytest_all.log
for f in gpurun_out/ty_bench_*.jsonl; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d['value'], d['roofline']['frac'], d['roofline']['ms_per_launch'], d['clocks'])" 2>/dev/null || head -c 300 $f; done
for f in gpurun_out/ty_flops_*.csv; do echo $f; grep -h "interval_kernel" $f | awk -F'","' '{print $(NF-2)" | "$NF}'; done
