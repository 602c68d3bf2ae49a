# ncu --set full of the cooperative scan on C2 (one sweep, 1e5 spin-one intervals)
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/s10_coop; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:scan_coop -s 1 -c 1 -o gpurun_out/s10_coop_c2 python tools/profile_run.py --workload C2 > $O/ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/s10_coop_c2.ncu-rep > $O/ncu_summary.txt 2>&1
cat $O/ncu_summary.txt; tail -3 $O/ncu.log
