"""The paper's accuracy experiment (§Evaluation of accuracy; Fig. 2, caption P:742-748) on the GPU path,
against the long-double oracle — SURVEY §8(f) NEXT #3.

Protocol, as printed:
* workload: Eq. neural_pulse — ω = 2π·700 kHz, Ω = 2π·1 kHz, Ω_p = 2π·70 Hz, a single-cycle sine pulse —
  driven for 100 ms with the 1 ms signal inside the run (t_p = 23.3 ms: reading R11), both spins, no quadratic
  shift (the equation has none; the spin-one exponentiator is Lie–Trotter τ = 24);
* every integration technique of P:702-704 — CF4, midpoint Euler, Heun Euler — with and without the rotating frame
  (P:705), over a ladder of time steps δt = Δt/L at Δt = 1 µs (K = 1e5 output samples);
* error: Eq. error, ε = (1/K)·sqrt(Σ_{k<K} Σ_m |ψ_k,m − ψ_k,m^baseline|²) (1/K outside the root as printed,
  reading R18), against a long-running baseline.  The paper's baseline is SciPy's `solve_ivp` (2.4 h); ours is the
  long-double oracle (CF4 + frame, the algorithm pinned to DOP853 in tests/test_oracle_pins.py [NS5]) at a step 4×
  (spin-one) / 8× (spin-half) finer than the finest one tested, so its own error is ≥ 256× below every error asserted
  on;
* errors above 1e-3 count as failed simulations; errors at the baseline's own accuracy are excluded (P:700:
  1e-11 for the paper's SciPy baseline, 1e-13 for ours — see FLOOR);
* execution time (Fig. 2b/2d): the device time of one ss_evaluate over a batch of 100 such simulations (dressing
  amplitude varied, the paper's device benchmark P:866-870), per simulation — batched so the time is the path's
  throughput, not launch latency.

Asserted (what the paper reports and the method fixes):
* CF4 is 4th order — error ÷ 10…24 per halving of δt (SURVEY [V6]) — and the Euler samplers 2nd order
  (÷ 3…6), on the rungs where both errors lie inside the window [FLOOR, 1e-3];
* the rotating frame makes every technique more accurate at every step where both runs pass ("4 orders");
* CF4 is more accurate than either Euler method at equal δt — ≥ 100× at the finest steps ("up to 3 orders");
* time to accuracy: every error ≤ 1e-7 an Euler run reaches, CF4 reaches in less device time;
* orders are read only on rungs that resolve the fastest oscillation of the integration frame (≥ 10 steps per period).
The table goes to $SPINSIM_EVIDENCE_DIR/fig2_accuracy.txt when that variable is set (profiles/r02/).
"""
import os

import numpy as np
import pytest
import torch

import workloads as W

pytestmark = pytest.mark.gpu

DT_OUT, T1 = 1e-6, 0.1
LADDER = [2, 4, 8, 16, 32]                  # δt = 500, 250, 125, 62.5, 31.25 ns
REF_L = {"half": 256, "one": 128}           # baseline δt = 3.9 / 7.8 ns
METHODS = ["cf4", "midpoint", "heun"]
# errors above 1e-3 are failed simulations; errors at the baseline's own accuracy are excluded.  The
# paper's SciPy baseline was good to 1e-11; ours (long-double oracle, step 4-8× finer) is limited by the GPU path's
# FP64 rounding, ≈ 3e-17 per interval, i.e. an RMS ≲ 1e-14 over K = 1e5 — so the floor is 1e-13.
FAIL, FLOOR = 1e-3, 1e-13
N_TIMED = 100                               # simulations per timed batch


def params():
    return W.neural_params(t_p=23.3e-3, omega_q=0.0)


@pytest.fixture(scope="module")
def study(orc):
    import paper_2204_05586_b200 as ss
    assert torch.cuda.is_available()
    out = {}
    for spin in ("half", "one"):
        d = 2 if spin == "half" else 3
        expo = "analytic" if spin == "half" else "lie_trotter"
        p = params()
        psi0 = W.basis_state(d)
        ref = orc.evaluate(spin, "cf4", expo, 24, True, "neural", sweep=p[None, :], t0=0.0, t1=T1,
                           dt_int=DT_OUT / REF_L[spin], dt_out=DT_OUT, psi0=psi0, want_unitaries=False)[0][0]
        # 100 simulations of the device benchmark: Ω varied ±10 %, simulation 0 is the measured one
        batch = np.repeat(p[None, :], N_TIMED, 0)
        batch[1:, 2] *= np.linspace(0.9, 1.1, N_TIMED - 1)
        sweep = torch.from_numpy(batch).cuda()
        psi = torch.from_numpy(W.basis_state(d, N_TIMED)).cuda()
        for method in METHODS:
            for frame in (True, False):
                sim = ss.Simulator(spin, method, expo, 24, frame, "fp64", "neural")
                for L in LADDER:
                    res = sim.evaluate(sweep, 0.0, T1, DT_OUT / L, DT_OUT, psi, want_unitaries=False)   # warm-up
                    sim.set_validation(False)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    res = sim.evaluate(sweep, 0.0, T1, DT_OUT / L, DT_OUT, psi, want_unitaries=False,
                                       out_states=res.state)
                    e1.record()
                    torch.cuda.synchronize()
                    sim.set_validation(True)
                    st = res.state[0].cpu().numpy()
                    K = st.shape[0] - 1
                    err = orc.rms_error(st[:K], ref[:K])          # Eq. error over k = 0 … K−1
                    out[(spin, method, frame, L)] = (err, float(np.abs(st - ref).max()),
                                                     e0.elapsed_time(e1) / N_TIMED)
    _write_table(out)
    return out


def _write_table(out):
    lines = [f"# Fig. 2 protocol (P:685-711): Eq. neural_pulse 100 ms, Δt = 1 µs (K = 1e5), RMS error (Eq. error) vs "
             f"the long-double oracle at δt = 1 µs/{REF_L['half']} (spin-half) / 1 µs/{REF_L['one']} (spin-one); "
             f"time = device ms per simulation in a batch of {N_TIMED}; '—' = failed (> 1e-3)"]
    for spin in ("half", "one"):
        lines.append(f"\n## spin-{spin}")
        lines.append(f"{'method':9s} {'frame':5s} " + " ".join(f"{'δt=' + format(1e3 / L, 'g') + 'ns':>12s}"
                                                              for L in LADDER) + "   ratio per halving")
        for method in METHODS:
            for frame in (True, False):
                errs = [out[(spin, method, frame, L)][0] for L in LADDER]
                ts = [out[(spin, method, frame, L)][2] for L in LADDER]
                cells = " ".join(f"{e:12.2e}" if e <= FAIL else f"{'—':>12s}" for e in errs)
                ratios = " ".join(f"{a / b:5.1f}" for a, b in zip(errs, errs[1:]))
                lines.append(f"{method:9s} {'on' if frame else 'off':5s} {cells}   {ratios}")
                lines.append(f"{'':9s} {'ms':5s} " + " ".join(f"{t:12.4f}" for t in ts))
    text = "\n".join(lines) + "\n"
    print(text)
    d = os.environ.get("SPINSIM_EVIDENCE_DIR")
    if d:
        os.makedirs(d, exist_ok=True)
        with open(os.path.join(d, "fig2_accuracy.txt"), "w") as f:
            f.write(text)


def _in_window(*errs):
    return all(FLOOR < e < FAIL for e in errs)


def _resolved(frame, dt):
    """The error expansion in powers of δt is asymptotic once the step resolves the fastest oscillation of the
    generator in the integration frame with ≥ 10 steps per period: in the lab frame the Larmor/RF frequency ω, in the
    rotating frame the counter-rotating component of the linear drive at 2ω (2Ω cos(ωt) Jx seen from a frame rotating
    at ω has components at 0 and 2ω)."""
    fast = (2.0 if frame else 1.0) * W.OMEGA_BIAS
    return fast * dt <= 2 * np.pi / 10


@pytest.mark.parametrize("spin", ["half", "one"])
@pytest.mark.parametrize("method", METHODS)
@pytest.mark.parametrize("frame", [True, False])
def test_convergence_order(study, spin, method, frame):
    lo, hi = (10.0, 24.0) if method == "cf4" else (3.0, 6.0)
    ratios = [study[(spin, method, frame, a)][0] / study[(spin, method, frame, b)][0]
              for a, b in zip(LADDER, LADDER[1:])
              if _in_window(study[(spin, method, frame, a)][0], study[(spin, method, frame, b)][0])
              and _resolved(frame, DT_OUT / a)]
    assert all(lo <= r <= hi for r in ratios), ratios
    if method == "cf4" or frame:
        assert ratios, "no resolved rung inside the paper's error window"
    else:                       # Euler in the lab frame: still failing (> 1e-3) at the coarser rungs (Fig. 2)
        assert study[(spin, method, frame, LADDER[2])][0] > FAIL


@pytest.mark.parametrize("spin", ["half", "one"])
@pytest.mark.parametrize("method", METHODS)
def test_rotating_frame_benefit(study, spin, method):
    for L in LADDER:
        on, off = study[(spin, method, True, L)][0], study[(spin, method, False, L)][0]
        if off < FAIL:
            assert on < off, (L, on, off)
    # at the finest step the benefit is large (the paper reports 4 orders on its own plots)
    on, off = study[(spin, method, True, LADDER[-1])][0], study[(spin, method, False, LADDER[-1])][0]
    assert off / on >= 100.0, (on, off)


@pytest.mark.parametrize("spin", ["half", "one"])
def test_cf4_beats_euler_at_equal_step(study, spin):
    for frame in (True, False):
        for L in LADDER:
            c = study[(spin, "cf4", frame, L)][0]
            for m in ("midpoint", "heun"):
                e = study[(spin, m, frame, L)][0]
                if e < FAIL:
                    assert c < e, (frame, L, m, c, e)
        c = study[(spin, "cf4", True, LADDER[-1])][0]
        for m in ("midpoint", "heun"):
            assert study[(spin, m, True, LADDER[-1])][0] / c >= 100.0


def _cf4_time_at(study, spin, err):
    """Device time CF4 + frame needs for RMS error `err`: log-log interpolation between the bracketing rungs of its
    time/error curve (error ∝ δt⁴, time ∝ 1/δt), None outside the measured range."""
    pts = [(study[(spin, "cf4", True, L)][0], study[(spin, "cf4", True, L)][2]) for L in LADDER]
    for (e0, t0), (e1, t1) in zip(pts, pts[1:]):
        if e1 <= err <= e0:
            f = np.log(e0 / err) / np.log(e0 / e1)
            return float(np.exp(np.log(t0) + f * np.log(t1 / t0)))
    return None


@pytest.mark.parametrize("spin", ["half", "one"])
def test_time_to_accuracy(study, spin):
    """CF4's accuracy outweighs its slower steps.  For every error ≤ 1e-7 an Euler run (frame on) reaches, CF4
    reaches the same error in less device time.  (Measured crossover: spin-one ≈ 1e-6 — a CF4 step
    costs two Lie–Trotter exponentials against the Euler step's one — spin-half above 4e-6.)"""
    checked = 0
    for m in ("midpoint", "heun"):
        for L in LADDER:
            e, t = study[(spin, m, True, L)][0], study[(spin, m, True, L)][2]
            if not (FLOOR < e <= 1e-7):
                continue
            tc = _cf4_time_at(study, spin, e)
            if tc is None:                            # below CF4's finest rung: CF4's finest is already more accurate
                tc = study[(spin, "cf4", True, LADDER[-1])][2]
                assert study[(spin, "cf4", True, LADDER[-1])][0] <= e
            assert tc < t, (m, L, e, t, tc)
            checked += 1
    assert checked >= 2
