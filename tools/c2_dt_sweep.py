"""The paper's spin-one benchmark (C2: Eq. neural_pulse + quadratic shift, 100 ms, one simulation) over the
time-step sweep BASELINE.json names (δt = 1 µs → 10 ns): fine steps/s of the whole hot path (interval kernel + scan)
per δt, CUDA-event timed after warm-up.  Also the paper's Fig. 4 device-benchmark workload (δt = 100 ns, 100
simulations varying the dressing amplitude) as one batched call.

    python tools/c2_dt_sweep.py > profiles/r01/c2_dt_sweep.txt
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_05586_b200 as ss  # noqa: E402
import workloads as W  # noqa: E402


def time_path(w, reps=5):
    sim = ss.Simulator(w.spin, w.method, w.expo, w.tau, w.frame, "fp64", w.field)
    sweep = torch.from_numpy(w.sweep).cuda()
    psi0 = torch.from_numpy(w.psi0).cuda()
    U = torch.empty((w.batch, w.K, 3, 3), dtype=torch.complex128, device="cuda")
    st = torch.empty((w.batch, w.K + 1, 3), dtype=torch.complex128, device="cuda")

    def step():
        sim.compute_unitaries(sweep, w.t0, w.t1, w.dt_int, w.dt_out, out=U)
        ss.scan_states(U, psi0, out=st)
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return ms, w.fine_steps / (ms * 1e-3)


def main():
    print("# C2: spin-one Eq. neural_pulse + ω_q, 100 ms, Δt = 1 µs (K = 1e5), Lie–Trotter τ = 24, frame on, FP64")
    print(f"{'δt':>8s} {'L':>4s} {'fine steps':>11s} {'ms/run':>9s} {'fine steps/s':>13s}")
    for L in (1, 2, 4, 10, 20, 40, 100):
        w = W.c2_neural(dt_int=1e-6 / L)
        ms, rate = time_path(w)
        print(f"{1e3 / L:6.0f}ns {L:4d} {w.fine_steps:11.3g} {ms:9.3f} {rate:13.3e}")
    w = W.c5_matrix("lie_trotter", batch=100).with_(sweep=W.c5_matrix("lie_trotter", batch=100).sweep)
    w = w.with_(sweep=w.sweep.copy())
    w.sweep[:, 6] = W.OMEGA_Q
    ms, rate = time_path(w)
    print(f"\n# paper Fig. 4 workload: 100 simulations × 100 ms at δt = 100 ns (dressing amplitude varied): "
          f"{ms:.2f} ms for all 100 ({ms / 100 * 1e3:.1f} µs per simulation), {rate:.3e} fine steps/s")


if __name__ == "__main__":
    main()
