export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for w in C3 C4 C2 G1; do
  timeout 300 python bench.py --workload $w --no-e2e --no-cpu-baseline --no-probe 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['value'], d['roofline']['frac'], d['roofline']['ms_per_launch'])"
done
timeout 300 python bench.py --workload C5 --expo analytic --no-e2e --no-cpu-baseline --no-probe 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C5an', d['value'], d['roofline']['frac'], d['roofline']['ms_per_launch'])"
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__inst_executed.sum,gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active
timeout 300 ncu --metrics $M --clock-control none -k regex:interval_kernel -s 1 -c 1 --csv python tools/profile_run.py --workload C4 --duration 0.1 2>&1 | grep interval_kernel | awk -F'","' '{print $(NF-2)" | "$NF}'
