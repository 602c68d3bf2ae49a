# one host-pipeline time chunk per wave (C2: 3 chunks) vs the wave pair: host-API tests + e2e A/B
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/s10_waves; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "host_api" 2>&1 | tail -2 > $O/pytest_host.log
for v in pair "" pair ""; do
  export SPINSIM_LIB=$PWD/paper_2204_05586_b200/libspinsim_b200${v:+.$v}.so
  timeout 300 python bench.py --workload C2 --no-cpu-baseline --no-probe --steps 20 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${v:-waves}', 'C2', d['value'], d['e2e']['value'], round(d['e2e']['value']/d['value'],4))" >> $O/ab.txt
done
cat $O/pytest_host.log $O/ab.txt
