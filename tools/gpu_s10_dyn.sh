# dynamic warp scheduling of the interval kernel for short problems (1-8 waves): all GPU tests + A/B on C2
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/s10_dyn; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3 > $O/pytest_gpu.log
for v in nodyn "" nodyn ""; do
  export SPINSIM_LIB=$PWD/paper_2204_05586_b200/libspinsim_b200${v:+.$v}.so
  timeout 300 python bench.py --workload C2 --no-cpu-baseline --no-probe --steps 20 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${v:-dyn}', 'C2', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['ms_per_launch'], d['e2e']['value'], d['gpu_launches'])" >> $O/ab.txt
done
unset SPINSIM_LIB
timeout 600 python tools/c2_dt_sweep.py > $O/c2_dt_sweep.txt 2>&1
cat $O/pytest_gpu.log $O/ab.txt; tail -12 $O/c2_dt_sweep.txt
