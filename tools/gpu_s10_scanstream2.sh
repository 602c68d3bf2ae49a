# scan stream only for the few-sweep tent (C4): host-API tests and the three e2e lines
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/s10_ss2; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "host_api" 2>&1 | tail -2 > $O/pytest_host.log
for w in C2 C4 C3; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline --no-probe 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['value'], d['e2e']['value'], round(d['e2e']['value']/d['value'],4))" >> $O/ab.txt
done
cat $O/pytest_host.log $O/ab.txt
