"""Interval-kernel rate of the paper's benchmark shape (one spin-one sweep, L = 10, split S = 2) against the number of
waves of interval threads: how much C2's partly empty last wave (1e5 intervals = 2.64 waves) costs.

    python tools/wave_probe.py > profiles/r02/<tag>/wave_probe.txt
"""
import sys, torch, numpy as np
sys.path.insert(0, '.')
import paper_2204_05586_b200 as ss, workloads as W
for K in (75776, 100000, 113664, 151552):
    w = W.c2_neural(duration=K * 1e-6)
    sim = ss.Simulator(w.spin, w.method, w.expo, w.tau, w.frame, "fp64", w.field)
    sw, p0 = torch.from_numpy(w.sweep).cuda(), torch.from_numpy(w.psi0).cuda()
    U = torch.empty((1, K, 3, 3), dtype=torch.complex128, device="cuda")
    for _ in range(3): sim.compute_unitaries(sw, w.t0, w.t1, w.dt_int, w.dt_out, out=U)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): sim.compute_unitaries(sw, w.t0, w.t1, w.dt_int, w.dt_out, out=U)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"K={K:7d} waves(S=2)={2*K/75776:5.2f} interval {ms*1e3:7.1f} us  {K*10/(ms*1e-3):.3e} steps/s")
