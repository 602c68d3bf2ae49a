# final r01 evidence: ncu full captures + executed-flop counters of the current kernels, bench lines, smoke
export PATH=/usr/local/cuda/bin:$PATH
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul_pred_on.sum,smsp__sass_thread_inst_executed_op_fadd_pred_on.sum,smsp__inst_executed.sum,gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active
timeout 300 ncu --metrics $M --clock-control none -k regex:interval_kernel -s 1 -c 1 --csv python tools/profile_run.py --workload C3 --batch 1024 > gpurun_out/f_flops_c3.csv 2>&1
timeout 300 ncu --metrics $M --clock-control none -k regex:interval_kernel -s 1 -c 1 --csv python tools/profile_run.py --workload C4 --duration 0.1 > gpurun_out/f_flops_c4.csv 2>&1
timeout 300 ncu --metrics $M --clock-control none -k regex:interval_kernel -s 1 -c 1 --csv python tools/profile_run.py --workload C5 --precision fp32 > gpurun_out/f_flops_c5_fp32.csv 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:interval_kernel -s 1 -c 1 -o gpurun_out/f_interval_c3 python tools/profile_run.py --workload C3 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:chain_kernel -s 1 -c 1 -o gpurun_out/f_chain_c3 python tools/profile_run.py --workload C3 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:interval_kernel -s 1 -c 1 -o gpurun_out/f_interval_c4 python tools/profile_run.py --workload C4 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/f_interval_c3.ncu-rep gpurun_out/f_chain_c3.ncu-rep gpurun_out/f_interval_c4.ncu-rep > gpurun_out/f_ncu_summary.txt 2>&1
timeout 600 python bench.py 2>&1 | tail -1 > gpurun_out/f_bench_default.jsonl
timeout 300 python bench.py --workload C4 2>&1 | tail -1 > gpurun_out/f_bench_c4.jsonl
timeout 300 python bench.py --workload C5 --precision fp32 --no-e2e --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/f_bench_c5_fp32.jsonl
timeout 300 python bench.py --workload C2 --no-e2e --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/f_bench_c2.jsonl
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-probe > /dev/null 2>&1
cat gpurun_out/f_ncu_summary.txt
grep -h "interval_kernel" gpurun_out/f_flops_*.csv | awk -F'","' '{print $5" | "$(NF-2)" | "$NF}'
for f in gpurun_out/f_bench_*.jsonl; do echo "$f: $(head -c 200 $f)"; done
