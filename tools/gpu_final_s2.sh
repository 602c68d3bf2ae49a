# session-2 evidence: all GPU tests, smoke, bench lines, reference arm, torchrun, launch list, ncu captures + counters
export PATH=/usr/local/cuda/bin:$PATH
O=${OUT:-gpurun_out/s2f}
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3 > $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py 2>&1 | tail -1 > $O/bench_default.jsonl
timeout 300 python bench.py --workload C4 2>&1 | tail -1 > $O/bench_c4.jsonl
timeout 300 python bench.py --workload C2 --no-cpu-baseline 2>&1 | tail -1 > $O/bench_c2.jsonl
timeout 300 python bench.py --workload C5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 > $O/bench_c5_lt_fp64.jsonl
timeout 300 python bench.py --workload C5 --precision fp32 --no-e2e --no-cpu-baseline 2>&1 | tail -1 > $O/bench_c5_lt_fp32.jsonl
timeout 300 python bench.py --workload C5 --expo analytic --no-e2e --no-cpu-baseline 2>&1 | tail -1 > $O/bench_c5_an_fp64.jsonl
timeout 300 python bench.py --workload G1 --no-e2e --no-cpu-baseline 2>&1 | tail -1 > $O/bench_g1.jsonl
timeout 300 python bench.py --workload C5 --expo analytic --precision fp32 --no-e2e --no-cpu-baseline 2>&1 | tail -1 > $O/bench_c5_an_fp32.jsonl
timeout 300 python bench.py --workload G1 --precision fp32 --no-e2e --no-cpu-baseline 2>&1 | tail -1 > $O/bench_g1_fp32.jsonl
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 1 --steps 3 --no-cpu-baseline 2>&1 | tail -1 > $O/bench_torchrun1.jsonl
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 2>&1 | tail -1 > $O/bench_reference.jsonl
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-probe > /dev/null 2>&1
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul_pred_on.sum,smsp__sass_thread_inst_executed_op_fadd_pred_on.sum,smsp__inst_executed.sum,gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active
timeout 300 ncu --metrics $M --clock-control none -k regex:interval_kernel -s 1 -c 1 --csv python tools/profile_run.py --workload C3 --batch 1024 > $O/flops_c3.csv 2>&1
timeout 300 ncu --metrics $M --clock-control none -k regex:interval_kernel -s 1 -c 1 --csv python tools/profile_run.py --workload C4 --duration 0.1 > $O/flops_c4.csv 2>&1
timeout 300 ncu --metrics $M --clock-control none -k regex:interval_kernel -s 1 -c 1 --csv python tools/profile_run.py --workload G1 --batch 1024 > $O/flops_g1.csv 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:interval_kernel -s 1 -c 1 -o $O/interval_c3 python tools/profile_run.py --workload C3 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:chain_kernel -s 1 -c 1 -o $O/chain_c3 python tools/profile_run.py --workload C3 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:interval_kernel -s 1 -c 1 -o $O/interval_c4 python tools/profile_run.py --workload C4 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:scan3_kernel -s 1 -c 1 -o $O/scan3_c5 python tools/profile_run.py --workload C5 > /dev/null 2>&1
python tools/ncu_summary.py $O/interval_c3.ncu-rep $O/chain_c3.ncu-rep $O/interval_c4.ncu-rep $O/scan3_c5.ncu-rep > $O/ncu_summary.txt 2>&1
rm -f $O/*.ncu-rep.tmp
cat $O/pytest_gpu.log $O/smoke.log | tail -8
for f in $O/bench_*.jsonl; do python -c "import json; d=json.load(open('$f')); print('$f', d['value'], d.get('ms_per_step'), d.get('roofline',{}).get('frac'), (d.get('e2e') or {}).get('value'), d.get('clocks',{}).get('sm_mhz'))" 2>/dev/null || head -c 300 $f; done
grep -E "^#|duration|fp64_pipe|dram_(read|write)" $O/ncu_summary.txt
