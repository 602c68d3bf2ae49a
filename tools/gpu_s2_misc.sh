# session 2: C5 matrix report, compute-sanitizer over the new kernel paths (su(3), SU(2)-form, specialised steps)
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_c5_matrix.py -q -s 2>&1 | tail -12
for tool in memcheck racecheck synccheck initcheck; do
  echo "== $tool"
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 99 python -m pytest tests/test_gpu_su3.py tests/test_gpu_parity.py -q -x \
     -k "su3_exponentiator_parity or su3_constant_parity or su3_euler or pulse_window or c1_rabi_parity or (scan_vs_sequential_chain and 3-255)" \
     -p no:cacheprovider 2>&1 | tail -3
  echo "exit=$?"
done > gpurun_out/sanitizer_s2.txt 2>&1
cat gpurun_out/sanitizer_s2.txt
