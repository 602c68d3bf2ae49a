# per-SASS-instruction execution / stall profile of the interval kernels (C4 spin-half, C3 spin-one)
export PATH=/usr/local/cuda/bin:$PATH
timeout 600 ncu --set full --import-source on --clock-control none -k regex:interval_kernel -s 1 -c 1 -o gpurun_out/sp_c4 python tools/profile_run.py --workload C4 --duration 0.1 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:interval_kernel -s 1 -c 1 -o gpurun_out/sp_c3 python tools/profile_run.py --workload C3 --batch 2048 > /dev/null 2>&1
for k in c4 c3; do
  ncu -i gpurun_out/sp_$k.ncu-rep --page source --csv --print-source sass > gpurun_out/sp_${k}_sass.csv 2>&1
done
ls -la gpurun_out/sp_*
head -3 gpurun_out/sp_c4_sass.csv | cut -c1-600
