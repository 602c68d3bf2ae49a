export PATH=/usr/local/cuda/bin:$PATH
for tool in memcheck racecheck synccheck initcheck; do
  echo "== $tool"
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 99 python -m pytest tests/test_gpu_magnus.py tests/test_gpu_parity.py -q -x \
     -k "magnus_bound_parity or c1_rabi_parity or c2_neural_parity_short or (scan_vs_sequential_chain and 3-255) or pulse_window" \
     -p no:cacheprovider 2>&1 | tail -3
  echo "exit=$?"
done > gpurun_out/sanitizer_s2b.txt 2>&1
cat gpurun_out/sanitizer_s2b.txt
