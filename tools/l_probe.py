"""Interval-kernel cost per interval against the fine steps per interval L (C3's spin-one Lie–Trotter sweep batch,
8192 sweeps, the same 8.2e7 fine steps at every L): fits time = K·(a + b·L) — b the throughput cost of a fine step,
a that of the once-per-interval work (prologue, frame exit, U_k store) — to say how much the per-interval code costs
at C3's L = 10.

    python tools/l_probe.py > profiles/r02/<tag>/l_probe.txt
"""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_2204_05586_b200 as ss  # noqa: E402
import workloads as W  # noqa: E402

B = 8192
rows = []
for L in (1, 2, 5, 10, 20, 40):
    dt_int = 100e-9
    dt_out = L * dt_int
    K = 10000 // L
    w = W.c3_batched(batch=B, duration=K * dt_out).with_(dt_int=dt_int, dt_out=dt_out)
    sim = ss.Simulator(w.spin, w.method, w.expo, w.tau, w.frame, "fp64", w.field)
    sw = torch.from_numpy(w.sweep).cuda()
    U = torch.empty((B, K, 3, 3), dtype=torch.complex128, device="cuda")
    for _ in range(2):
        sim.compute_unitaries(sw, w.t0, w.t1, w.dt_int, w.dt_out, out=U)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        sim.compute_unitaries(sw, w.t0, w.t1, w.dt_int, w.dt_out, out=U)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    steps = B * K * L
    rows.append((L, B * K, ms))
    print(f"L={L:3d} K={K:6d} intervals={B*K:9d} interval kernel {ms:9.3f} ms  {steps/(ms*1e-3):.4e} fine steps/s",
          flush=True)
    del U
    torch.cuda.empty_cache()
A = np.array([[n, n * L] for L, n, _ in rows], dtype=float)
y = np.array([ms for _, _, ms in rows])
(a, b), *_ = np.linalg.lstsq(A, y, rcond=None)
print(f"fit: per interval a = {a*1e6:.2f} ns-equivalent, per fine step b = {b*1e6:.2f} ns-equivalent "
      f"(device-wide throughput); at L = 10 the per-interval work is {a/(a+10*b):.3f} of the kernel")
