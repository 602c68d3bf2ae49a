# the staged cooperative scan's bounds against the oracle chain
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/s10_stagetest; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "staging_boundary" 2>&1 | tail -4 > $O/pytest.log
cat $O/pytest.log
