# staged cooperative scan: 128 vs 256 CTAs per sweep (two staged CTAs per SM) on C2 and C1-size problems
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/s10_cps; mkdir -p $O
for v in "" cps256 "" cps256; do
  export SPINSIM_LIB=$PWD/paper_2204_05586_b200/libspinsim_b200${v:+.$v}.so
  timeout 300 python bench.py --workload C2 --no-cpu-baseline --no-probe --no-e2e --steps 20 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${v:-cps128}', 'C2', d['value'], d['ms_per_step'], d.get('scan', {}).get('ms_per_launch'))" >> $O/ab.txt
done
export SPINSIM_LIB=$PWD/paper_2204_05586_b200/libspinsim_b200.cps256.so
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "c2 or c1 or grid_edge or host_api" 2>&1 | tail -2 > $O/pytest_cps256.log
cat $O/ab.txt $O/pytest_cps256.log
