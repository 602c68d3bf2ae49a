# Final round-2 evidence: gpu_evidence.sh (tests, smoke, default + reference bench, launch list, ncu summaries, executed
# flops, SASS), gpu_bench_lines.sh (every bench line, shard emulations, C2 dt sweep, scan-stress), and the scan3
# ring-depth variants on the scan paths.   gpurun -- 'bash tools/gpu_final.sh TAG'
set -u
T=${1:-final}
bash tools/gpu_evidence.sh ${T} all > gpurun_out/${T}_evidence.log 2>&1
bash tools/gpu_bench_lines.sh ${T}_lines > gpurun_out/${T}_lines.log 2>&1
for v in s3n2 s3n3; do
  if [ -f paper_2204_05586_b200/libspinsim_b200.$v.so ]; then
    SPINSIM_LIB=$PWD/paper_2204_05586_b200/libspinsim_b200.$v.so timeout 600 python tools/scan_paths.py > gpurun_out/${T}/scan_paths_$v.txt 2>&1
  fi
done
timeout 600 python tools/scan_paths.py > gpurun_out/${T}/scan_paths.txt 2>&1
tail -5 gpurun_out/${T}/pytest_gpu.log; cat gpurun_out/${T}_lines.log | tail -30
