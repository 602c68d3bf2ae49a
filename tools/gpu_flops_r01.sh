# executed FP64/FP32 flop counters (thread-level SASS counts) for the interval kernel on C3 (subset) and C4 (prefix)
export PATH=/usr/local/cuda/bin:$PATH
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul_pred_on.sum,smsp__sass_thread_inst_executed_op_fadd_pred_on.sum,smsp__inst_executed.sum,gpu__time_duration.sum
timeout 300 ncu --metrics $M --clock-control none -k regex:interval_kernel -s 1 -c 1 --csv python tools/profile_run.py --workload C3 --batch 1024 > gpurun_out/r01_flops_c3.csv 2>&1
timeout 300 ncu --metrics $M --clock-control none -k regex:interval_kernel -s 1 -c 1 --csv python tools/profile_run.py --workload C4 --duration 0.1 > gpurun_out/r01_flops_c4.csv 2>&1
timeout 300 ncu --metrics $M --clock-control none -k regex:interval_kernel -s 1 -c 1 --csv python tools/profile_run.py --workload C5 --precision fp32 > gpurun_out/r01_flops_c5_fp32.csv 2>&1
grep -h "interval_kernel" gpurun_out/r01_flops_*.csv | awk -F'","' '{print $5" | "$(NF-2)" | "$NF}'
