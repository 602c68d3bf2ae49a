# compute-sanitizer over the scan (decoupled look-back, mbarriers, TMA) and interval kernels
export PATH=/usr/local/cuda/bin:$PATH
for tool in memcheck racecheck synccheck initcheck; do
  echo "== $tool"
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 99 python -m pytest tests/test_gpu_parity.py -q -x \
     -k "scan_vs_sequential_chain and (3-255 or 4100-37 or 5-1031) or fused_spin and 3-1031 or c1_rabi_parity" \
     -p no:cacheprovider 2>&1 | tail -4
  echo "exit=$?"
done
