"""Accuracy-vs-time-step study in the shape of the paper's Fig. 2 (§accuracy), run on the GPU.

For spin-half and spin-one (Lie–Trotter), each integration method (CF4, midpoint Euler, Heun Euler) with and
without the rotating frame is run over a ladder of fine steps δt = Δt/L, and its RMS error (Eq. error, P:689,
1/K outside the root as printed — reading R18) and max-abs amplitude error are taken against a reference: CF4 with the
frame at δt = 1 ns (its own agreement with the long-double oracle at that δt is asserted by tests/test_gpu_fullsize.py).
The workload is Eq. neural_pulse over a 1 ms window that contains the 1 ms signal pulse (t_p = 0.2 ms).

    python tools/accuracy_study.py > profiles/r01/accuracy_study.txt

Reported per configuration: error at each δt, the error ratio per halving of δt (4th order → ≈16, 2nd order → ≈4) and
the GPU time of the interval kernel.  Errors above 1e-3 are "failed" as in P:699.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_05586_b200 as ss  # noqa: E402
import workloads as W  # noqa: E402


def rms_error(a: np.ndarray, b: np.ndarray) -> float:
    """Eq. error: (1/K) sqrt(Σ_k Σ_m |ψ − ψ_ref|²) over the K output samples."""
    K = a.shape[0] - 1
    return float(np.sqrt(np.sum(np.abs(a[:-1] - b[:-1]) ** 2)) / K)


def run(spin, method, frame, L, t1=1e-3):
    expo = "analytic" if spin == "half" else "lie_trotter"
    p = W.neural_params(t_p=0.2e-3, omega_q=W.OMEGA_Q if spin == "one" else 0.0)
    sim = ss.Simulator(spin, method, expo, 24, frame, "fp64", "neural")
    sweep = torch.from_numpy(p[None, :]).cuda()
    psi0 = torch.from_numpy(W.basis_state(2 if spin == "half" else 3)).cuda()
    dt_out = 1e-6
    U = sim.compute_unitaries(sweep, 0.0, t1, dt_out / L, dt_out)          # warm
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    U = sim.compute_unitaries(sweep, 0.0, t1, dt_out / L, dt_out)
    e1.record()
    st = ss.scan_states(U, psi0)
    torch.cuda.synchronize()
    return st[0].cpu().numpy(), e0.elapsed_time(e1)


def main():
    Ls = [1, 2, 4, 8, 16, 32, 64]
    for spin in ("half", "one"):
        ref, _ = run(spin, "cf4", True, 1000)
        print(f"## spin-{spin}: Eq. neural_pulse, 1 ms window with the signal pulse, Δt = 1 µs (K = 1000); "
              f"reference CF4 + frame at δt = 1 ns")
        print(f"{'method':9s} {'frame':5s} " + " ".join(f"{'δt=' + format(1e3 / L, 'g') + 'ns':>11s}" for L in Ls)
              + "   halving ratios (RMS)")
        for method in ("cf4", "midpoint", "heun"):
            for frame in (True, False):
                errs, maxs, times = [], [], []
                for L in Ls:
                    st, ms = run(spin, method, frame, L)
                    errs.append(rms_error(st, ref))
                    maxs.append(float(np.abs(st - ref).max()))
                    times.append(ms)
                ratios = [a / b for a, b in zip(errs, errs[1:]) if b > 0]
                cells = " ".join(f"{e:11.2e}" if e <= 1e-3 else f"{'failed':>11s}" for e in errs)
                print(f"{method:9s} {'on' if frame else 'off':5s} {cells}   "
                      + " ".join(f"{r:5.1f}" for r in ratios))
                print(f"{'':9s} {'max':5s} " + " ".join(f"{m:11.2e}" for m in maxs) +
                      "   kernel ms: " + " ".join(f"{t:.3f}" for t in times))
        print()


if __name__ == "__main__":
    main()
