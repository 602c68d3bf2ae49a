# general spin-one: su3 + randomised parity, executed-flop counters and one ncu --set full capture of the G1 kernel
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_gpu_su3.py tests/test_gpu_random_parity.py -q 2>&1 | tail -4 > gpurun_out/su3b_pytest.log
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__inst_executed.sum,gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active
timeout 300 ncu --metrics $M --clock-control none -k regex:interval_kernel -s 1 -c 1 --csv python tools/profile_run.py --workload G1 --batch 1024 > gpurun_out/su3b_flops_g1.csv 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:interval_kernel -s 1 -c 1 -o gpurun_out/su3b_interval_g1 python tools/profile_run.py --workload G1 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/su3b_interval_g1.ncu-rep > gpurun_out/su3b_ncu_summary.txt 2>&1
timeout 300 python bench.py --workload G1 --no-e2e 2>&1 | tail -1 > gpurun_out/su3b_bench_g1.jsonl
cat gpurun_out/su3b_pytest.log gpurun_out/su3b_ncu_summary.txt
grep -h "interval_kernel" gpurun_out/su3b_flops_g1.csv | awk -F'","' '{print $(NF-2)" | "$NF}'
head -c 400 gpurun_out/su3b_bench_g1.jsonl
