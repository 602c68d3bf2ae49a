export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for w in C4 C2 C3; do
  timeout 300 python bench.py --workload $w --no-cpu-baseline --no-probe $( [ $w = C4 ] || echo --no-e2e ) 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['value'], d['roofline']['frac'], d['roofline']['ms_per_launch'], d.get('e2e'))"
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --workload C4 --gpus 2 --share-gpu --dist-backend gloo --no-cpu-baseline --steps 3 2>&1 | tail -1 | head -c 300; echo
