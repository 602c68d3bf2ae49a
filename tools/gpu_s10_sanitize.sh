# compute-sanitizer over the session-4 host-pipeline paths (wave pair, C4-style tent with a scan stream)
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/s10_san; mkdir -p $O
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "wave_pair or matches_device" > $O/memcheck.txt 2>&1
tail -5 $O/memcheck.txt
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "wave_pair and 1" > $O/racecheck.txt 2>&1
tail -5 $O/racecheck.txt
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -c "
import numpy as np, paper_2204_05586_b200 as ss, workloads as W
w = W.c4_long(duration=0.02)
sim = ss.Simulator(w.spin, w.method, w.expo, w.tau, w.frame, 'fp64', w.field)
print(sim.host_chunk_plan(w.t0, w.t1, w.dt_int, w.dt_out, 1, 6))
st, U = sim.evaluate_host(w.sweep, w.t0, w.t1, w.dt_int, w.dt_out, w.psi0, want_unitaries=True, n_chunks=6)
print('norm drift', float(np.abs(np.linalg.norm(st, axis=-1) - 1).max()))
" > $O/memcheck_c4tent.txt 2>&1
tail -5 $O/memcheck_c4tent.txt
