"""Time the interval kernel on a C4 partition slice (one rank's share at N ranks) for the split the library picks."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_05586_b200 as ss  # noqa: E402
import workloads as W  # noqa: E402

w = W.c4_long()
sim = ss.Simulator(w.spin, w.method, w.expo, w.tau, w.frame, "fp64", w.field)
sweep = torch.from_numpy(w.sweep).cuda()
for n_ranks in (1, 2, 4, 8):
    kc = w.K // n_ranks
    U = torch.empty((1, kc, 2, 2), dtype=torch.complex128, device="cuda")
    for _ in range(2):
        sim.compute_unitaries(sweep, w.t0, w.t1, w.dt_int, w.dt_out, k_begin=0, k_count=kc, out=U)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(3):
        sim.compute_unitaries(sweep, w.t0, w.t1, w.dt_int, w.dt_out, k_begin=0, k_count=kc, out=U)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"{os.path.basename(ss._lib.LIB_PATH)} N={n_ranks} k_count={kc}: {ms:.3f} ms ({kc * w.L / (ms * 1e-3):.3e} fine steps/s per rank)")
