# ncu captures for profiles/r01 (run under gpurun; one GPU)
export PATH=/usr/local/cuda/bin:$PATH
set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:interval_kernel -s 1 -c 1 -o gpurun_out/r01_interval_c3 python tools/profile_run.py --workload C3 > gpurun_out/r01_ncu_interval_c3.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:chain_kernel -s 1 -c 1 -o gpurun_out/r01_chain_c3 python tools/profile_run.py --workload C3 > gpurun_out/r01_ncu_chain_c3.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:scan2 -s 1 -c 1 -o gpurun_out/r01_scan2_c5 python tools/profile_run.py --workload C5 > gpurun_out/r01_ncu_scan2_c5.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:interval_kernel -s 1 -c 1 -o gpurun_out/r01_interval_c4 python tools/profile_run.py --workload C4 > gpurun_out/r01_ncu_interval_c4.log 2>&1
python tools/ncu_summary.py gpurun_out/r01_interval_c3.ncu-rep gpurun_out/r01_chain_c3.ncu-rep gpurun_out/r01_scan2_c5.ncu-rep gpurun_out/r01_interval_c4.ncu-rep > gpurun_out/r01_ncu_summary.txt 2>&1
cat gpurun_out/r01_ncu_summary.txt
