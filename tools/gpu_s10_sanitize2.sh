# compute-sanitizer memcheck over C4's time tent with the scan stream (full 1 s sweep, 6 chunks)
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/s10_san; mkdir -p $O
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -c "
import numpy as np, paper_2204_05586_b200 as ss, workloads as W
w = W.c4_long()
sim = ss.Simulator(w.spin, w.method, w.expo, w.tau, w.frame, 'fp64', w.field)
print(sim.host_chunk_plan(w.t0, w.t1, w.dt_int, w.dt_out, 1, 6))
st, U = sim.evaluate_host(w.sweep, w.t0, w.t1, w.dt_int, w.dt_out, w.psi0, want_unitaries=True, n_chunks=6)
print('norm drift', float(np.abs(np.linalg.norm(st, axis=-1) - 1).max()))
" > $O/memcheck_c4tent.txt 2>&1
tail -5 $O/memcheck_c4tent.txt
