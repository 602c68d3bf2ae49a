# tridiagonalised su(3) path: compute-sanitizer, G1 full-length sweeps vs the oracle, spill traffic of C3/G1
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/su3v; mkdir -p $O
for tool in memcheck initcheck; do
  echo "== $tool"
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 99 python -m pytest tests/test_gpu_su3.py -q -x \
     -k "su3_exponentiator_parity or su3_constant_parity or fp32" -p no:cacheprovider 2>&1 | tail -2
  echo "exit=$?"
done > $O/sanitizer.txt 2>&1
SPINSIM_LONG=1 timeout 900 python -m pytest tests/test_gpu_long_verification.py -q -s -k "g1 or c3" 2>&1 | grep -E "G1|C3|passed|failed" > $O/long_verification.txt
M=l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum,l1tex__t_bytes_pipe_lsu_mem_local_op_st.sum,smsp__inst_executed.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active
timeout 300 ncu --metrics $M --clock-control none -k regex:interval_kernel -s 1 -c 1 --csv python tools/profile_run.py --workload C3 --batch 1024 > $O/local_c3.csv 2>&1
cat $O/sanitizer.txt $O/long_verification.txt
grep -E "local|fp64|inst_executed" $O/local_c3.csv | awk -F'","' '{print $(NF-2), $NF}'
