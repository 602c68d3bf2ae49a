"""GPU test + report for BASELINE config 5: the spin-one analytic-vs-Lie–Trotter and FP32-vs-FP64 accuracy/throughput matrix at the fixed
100 ms workload (Eq. neural_pulse as printed, ω_q = 0, δt = 100 ns, Δt = 1 µs) against the CPU oracle.

* accuracy: one simulation (C5 accuracy variant), max |ψ_gpu − ψ_oracle| over all 1e5 + 1 states against the
  long-double oracle of the SAME exponentiator, and against the other exponentiator's oracle (analytic ↔ LT: the
  two methods differ only by roundoff here, SURVEY [V19]);
* throughput: the 100-sweep C5 batch, whole hot path (interval kernel + scan), CUDA events after warm-up;
* the oracle's own CPU time for the single simulation (double instantiation, all host cores), for context.

    python -m pytest tests/test_gpu_c5_matrix.py -m gpu -s      # table on stdout and in gpurun_out/c5_matrix.txt

(A test, not a tool: only tests/, smoke() and bench.py's baseline legs may run the oracle.)  The assertions are the
north-star bars: 1e-10 in FP64 and 1e-4 in FP32 against the oracle of the same exponentiator.
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pytest  # noqa: E402

import oracle  # noqa: E402
import paper_2204_05586_b200 as ss  # noqa: E402
import workloads as W  # noqa: E402

pytestmark = pytest.mark.gpu


def gpu_states(w, precision):
    sim = ss.Simulator(w.spin, w.method, w.expo, w.tau, w.frame, precision, w.field)
    res = sim.evaluate(torch.from_numpy(w.sweep).cuda(), w.t0, w.t1, w.dt_int, w.dt_out,
                       torch.from_numpy(w.psi0).cuda(), want_unitaries=False)
    torch.cuda.synchronize()
    return res.state.cpu().numpy()


def throughput(w, precision, reps=5):
    sim = ss.Simulator(w.spin, w.method, w.expo, w.tau, w.frame, precision, w.field)
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


def test_c5_matrix():
    lines = []
    out = lines.append
    ref = {}
    cpu_s = {}
    for expo in ("analytic", "lie_trotter"):
        w = W.c5_matrix(expo, batch=1)
        t = time.time()
        ref[expo], _ = oracle.evaluate(w.spin, w.method, w.expo, w.tau, w.frame, w.field, sweep=w.sweep, t0=w.t0,
                                       t1=w.t1, dt_int=w.dt_int, dt_out=w.dt_out, psi0=w.psi0, want_unitaries=False)
        cpu_s[expo] = time.time() - t
    out("# C5: spin-one Eq. neural_pulse as printed (ω_q = 0), 100 ms, δt = 100 ns, Δt = 1 µs, τ = 24, frame on")
    out(f"# oracle (long double, {os.cpu_count()} host threads) for one simulation: analytic {cpu_s['analytic']:.1f} s,"
          f" Lie–Trotter {cpu_s['lie_trotter']:.1f} s")
    out(f"# oracle analytic vs oracle Lie–Trotter: max |Δψ| = {np.abs(ref['analytic'] - ref['lie_trotter']).max():.2e}")
    out(f"{'exponentiator':>13s} {'precision':>9s} {'max|ψ−oracle|':>14s} {'vs other expo':>14s} "
          f"{'100-sweep ms':>13s} {'fine steps/s':>13s}")
    for expo in ("analytic", "lie_trotter"):
        other = "lie_trotter" if expo == "analytic" else "analytic"
        for prec in ("fp64", "fp32"):
            w1 = W.c5_matrix(expo, batch=1)
            st = gpu_states(w1, prec)
            e_same = np.abs(st - ref[expo]).max()
            e_other = np.abs(st - ref[other]).max()
            ms, rate = throughput(W.c5_matrix(expo, batch=100), prec)
            out(f"{expo:>13s} {prec:>9s} {e_same:14.2e} {e_other:14.2e} {ms:13.3f} {rate:13.3e}")
            assert e_same <= (1e-10 if prec == "fp64" else 1e-4), (expo, prec, e_same)
    text = "\n".join(lines)
    print(text)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if os.path.isdir(os.path.join(root, "gpurun_out")):
        with open(os.path.join(root, "gpurun_out", "c5_matrix.txt"), "w") as f:
            f.write(text + "\n")
