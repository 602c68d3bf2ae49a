export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out/su3t
timeout 900 python -m pytest tests -m gpu -q -x -k "su3 or g1 or G1 or random_parity or magnus" 2>&1 | tail -5 > gpurun_out/su3t/pytest.log
for i in 1 2; do
timeout 300 python bench.py --workload G1 --no-e2e --no-cpu-baseline --no-probe --steps 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('G1', d['value'], d['roofline']['ms_per_launch'])"
timeout 300 python bench.py --workload G1 --precision fp32 --no-e2e --no-cpu-baseline --no-probe --steps 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('G1f32', d['value'], d['roofline']['ms_per_launch'])"
done
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__inst_executed.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum,l1tex__t_bytes_pipe_lsu_mem_local_op_st.sum
timeout 300 ncu --metrics $M --clock-control none -k regex:interval_kernel -s 1 -c 1 --csv python tools/profile_run.py --workload G1 --batch 1024 > gpurun_out/su3t/flops_g1.csv 2>&1
grep -E "op_d|fp64|inst_executed.sum|local" gpurun_out/su3t/flops_g1.csv | awk -F'","' '{print $(NF-2), $NF}'
cat gpurun_out/su3t/pytest.log
