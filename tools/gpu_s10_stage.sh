# cooperative scan with the CTA's operators staged in shared memory (one bulk copy) vs the L2 path: GPU tests + A/B
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/s10_stage; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > $O/pytest_gpu.log
cat $O/pytest_gpu.log
for v in nostage "" nostage ""; do
  export SPINSIM_LIB=$PWD/paper_2204_05586_b200/libspinsim_b200${v:+.$v}.so
  for w in C2 C4; do
  timeout 300 python bench.py --workload $w --no-cpu-baseline --no-probe --steps 20 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${v:-staged}', '$w', d['value'], d['ms_per_step'], d.get('scan', {}).get('ms_per_launch'), d.get('exchange_and_scan_ms'), d['e2e']['value'])" >> $O/ab.txt
  done
done
unset SPINSIM_LIB
timeout 300 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_parity.py -m gpu -q -k "c2_neural_parity_short or c1_rabi or grid_edge" > $O/memcheck.txt 2>&1
timeout 300 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py -m gpu -q -k "c2_neural_parity_short" > $O/racecheck.txt 2>&1
timeout 300 ncu --set full --clock-control none -k regex:scan_coop -s 1 -c 1 -o gpurun_out/s10_coop_staged python tools/profile_run.py --workload C2 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/s10_coop_staged.ncu-rep > $O/ncu_summary.txt 2>&1
cat $O/ab.txt; tail -2 $O/memcheck.txt $O/racecheck.txt; head -16 $O/ncu_summary.txt
