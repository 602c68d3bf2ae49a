export PATH=/usr/local/cuda/bin:$PATH
for v in "" t32 t32c16 t64c4 t128c4; do
  export SPINSIM_LIB=$PWD/paper_2204_05586_b200/libspinsim_b200${v:+.$v}.so
  timeout 300 python bench.py --steps 3 --no-e2e --no-cpu-baseline --no-probe 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${v:-base}', d['value'], d['scan'])"
done
export SPINSIM_LIB=$PWD/paper_2204_05586_b200/libspinsim_b200.t32.so
timeout 300 python -m pytest tests -m gpu -q -x -k "scan or c3" 2>&1 | tail -1
