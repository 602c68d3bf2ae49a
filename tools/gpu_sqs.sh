export PATH=/usr/local/cuda/bin:$PATH
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -2
SPINSIM_LONG=1 timeout 900 python -m pytest tests/test_gpu_long_verification.py -q -s -k c3 2>&1 | grep -E "C3|passed|failed"
for v in "" f1; do
  export SPINSIM_LIB=$PWD/paper_2204_05586_b200/libspinsim_b200${v:+.$v}.so
  for w in C3 C2; do
    timeout 300 python bench.py --workload $w --no-e2e --no-cpu-baseline --no-probe 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${v:-f2}', '$w', d['value'], d['roofline']['ms_per_launch'])"
  done
  timeout 300 python bench.py --workload C5 --precision fp32 --no-e2e --no-cpu-baseline --no-probe 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${v:-f2}', 'C5f32', d['value'], d['roofline']['ms_per_launch'])"
done
unset SPINSIM_LIB
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__inst_executed.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active
timeout 300 ncu --metrics $M --clock-control none -k regex:interval_kernel -s 1 -c 1 --csv python tools/profile_run.py --workload C3 --batch 1024 2>&1 | grep interval_kernel | awk -F'","' '{print $(NF-2)" | "$NF}'
