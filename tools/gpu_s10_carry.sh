# time-chunk carry by a gather kernel vs cudaMemcpy2DAsync: host-API tests + C3/C4/C2 e2e A/B
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/s10_carry; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "host_api" 2>&1 | tail -2 > $O/pytest_host.log
for v in memcpy2d "" memcpy2d ""; do
  export SPINSIM_LIB=$PWD/paper_2204_05586_b200/libspinsim_b200${v:+.$v}.so
  for w in C3 C4; do
    timeout 600 python bench.py --workload $w --no-cpu-baseline --no-probe 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${v:-gather}', '$w', d['value'], d['e2e']['value'], round(d['e2e']['value']/d['value'],4))" >> $O/ab.txt
  done
done
cat $O/pytest_host.log $O/ab.txt
