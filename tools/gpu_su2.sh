export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/su2_pytest.log
timeout 300 python bench.py --workload C4 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/su2_bench_c4.jsonl
timeout 300 python bench.py --workload C4 --precision fp32 --no-e2e --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/su2_bench_c4_fp32.jsonl
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__inst_executed.sum,gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
timeout 300 ncu --metrics $M --clock-control none -k regex:interval_kernel -s 1 -c 1 --csv python tools/profile_run.py --workload C4 --duration 0.1 > gpurun_out/su2_flops_c4.csv 2>&1
cat gpurun_out/su2_pytest.log
for f in gpurun_out/su2_bench_*.jsonl; do python -c "import json; d=json.load(open('$f')); print('$f', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['ms_per_launch'], d.get('e2e'))" 2>/dev/null || head -c 400 $f; done
grep -h "interval_kernel" gpurun_out/su2_flops_c4.csv | awk -F'","' '{print $(NF-2)" | "$NF}'
