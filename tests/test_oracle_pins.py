"""Pins for the CPU oracle (oracle/): each check ties the oracle to something OTHER than itself — the paper's
printed values, closed forms, scipy.linalg.expm / scipy.integrate on textbook matrices built here, brute force,
invariants.  The five north-star pins (BASELINE.json) are marked [NS1]…[NS5].  Citations: P:<line> = PAPER.md.

These run without a GPU (`-m "not gpu"`).
"""
import decimal
import json
import math
import os

import numpy as np
import pytest
import scipy.integrate as si
import scipy.linalg as sl

import workloads as W

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))

# ---- textbook operators, built here independently of the oracle ------------------------------------------
SX = np.array([[0, 1], [1, 0]], complex)
SY = np.array([[0, -1j], [1j, 0]], complex)
SZ = np.diag([1.0, -1.0]).astype(complex)
R2 = 1 / math.sqrt(2)
J1X = R2 * np.array([[0, 1, 0], [1, 0, 1], [0, 1, 0]], complex)
J1Y = R2 * np.array([[0, -1j, 0], [1j, 0, -1j], [0, 1j, 0]], complex)
J1Z = np.diag([1.0, 0.0, -1.0]).astype(complex)
Q = np.diag([1.0, -2.0, 1.0]).astype(complex) / 3


def ops(spin):
    if spin == "half":
        return SX / 2, SY / 2, SZ / 2, np.zeros((2, 2), complex)
    return J1X, J1Y, J1Z, Q


def H_of(spin, f):
    jx, jy, jz, q = ops(spin)
    return f[0] * jx + f[1] * jy + f[2] * jz + f[3] * q


def run(orc, w, **kw):
    return orc.evaluate(w.spin, w.method, w.expo, w.tau, w.frame, w.field, sweep=w.sweep, t0=w.t0, t1=w.t1,
                        dt_int=w.dt_int, dt_out=w.dt_out, psi0=w.psi0, **kw)


# ---- operator algebra sanity (the test's own matrices, so the pins below stand on solid ground) -----------
def test_textbook_operators():
    for spin, j in (("half", 0.5), ("one", 1.0)):
        jx, jy, jz, _ = ops(spin)
        assert np.allclose(jx @ jy - jy @ jx, 1j * jz, atol=1e-15)
        assert np.allclose(jx @ jx + jy @ jy + jz @ jz, j * (j + 1) * np.eye(len(jz)), atol=1e-15)
    assert np.allclose(Q, J1Z @ J1Z - 2 / 3 * np.eye(3), atol=1e-15)          # P:181 "Q ∝ Jz²"
    assert np.allclose(np.diag(Q) * 3, GOLD["quadrupole_Q_diag"]["diag_times_3"])


# ---- CF4 constants vs 50-digit decimal evaluation ---------------------------------------------
def _dec(expr):
    decimal.getcontext().prec = 60
    s3 = decimal.Decimal(3).sqrt()
    return float(expr(s3))        # float(Decimal) is correctly rounded


def test_cf4_constants_correctly_rounded(orc):
    c = orc.constants()
    assert c["g1"] == _dec(lambda s3: (1 - 1 / s3) / 2)
    assert c["g2"] == _dec(lambda s3: (1 + 1 / s3) / 2)
    assert c["w_plus"] == _dec(lambda s3: (3 + 2 * s3) / 12)
    assert c["w_minus"] == _dec(lambda s3: (3 - 2 * s3) / 12)
    assert c["w_minus"] < 0
    assert c["w_plus"] + c["w_minus"] == 0.5
    for case in GOLD["gauss_times"]["cases"]:
        t1 = case["t"] + c["g1"] * case["dt"]
        t2 = case["t"] + c["g2"] * case["dt"]
        # SPEC prints the leading digits ("0.7886751345…", truncated or rounded)
        assert abs(t1 - case["t1"]) < 10 ** -case["digits"]
        assert abs(t2 - case["t2"]) < 10 ** -case["digits"]
    assert round(c["w_plus"], 4) == GOLD["cf4_weight_example"]["h1_x"]


def test_time_grid(orc):
    K, L, dt = orc.plan(0.0, 0.1, 100e-9, 1e-6)
    assert (K, L) == (100000, 10) and dt == 1e-6 / 10
    g = orc.grid(0.0, 1e-6, dt, 12345, 7)
    assert g["t_k"] == 12345 * 1e-6
    assert g["off1"] < g["off_mid"] < g["off2"] < 8 * dt
    assert abs((g["off1"] + g["off2"]) / 2 - 7.5 * dt) < 1e-21
    with pytest.raises(ValueError):
        orc.plan(0.0, 0.1, 300e-9, 1e-6)          # L not integral (reading R10)
    with pytest.raises(ValueError):
        orc.plan(0.0, 0.10005e0 + 3e-7, 100e-9, 1e-6)


# ---- exponentiators ----------------------------------------------------------------------------------------
def test_su2_closed_form_vs_expm(orc):
    a = W.random_exponent_args(4000, 1.0, seed=1)
    U = orc.exponentiate("half", a)
    ref = np.array([sl.expm(-1j * H_of("half", x)) for x in a])
    assert np.abs(U - ref).max() < 1e-14
    # S:130-133 examples
    assert np.abs(orc.exponentiate("half", [[0, 0, 0, 0]])[0] - np.eye(2)).max() == 0
    th = 0.7
    assert np.allclose(orc.exponentiate("half", [[0, 0, th, 0]])[0],
                       np.diag([np.exp(-0.5j * th), np.exp(0.5j * th)]), atol=1e-16)
    g = np.array(GOLD["expm_su2_examples"]["minus_i_sigma_x"], float)
    assert np.allclose(orc.exponentiate("half", [[np.pi, 0, 0, 0]])[0], g[..., 0] + 1j * g[..., 1], atol=1e-16)


def _residual_series(X, terms=30):
    """exp(−iX) − I by its Taylor series without ever forming I + … (no cancellation)."""
    acc = np.zeros_like(X)
    term = np.eye(len(X), dtype=complex)
    for k in range(1, terms):
        term = term @ (-1j * X) / k
        acc = acc + term
    return acc


def test_trotter_factor_residual_vs_leapfrog_product(orc):
    """I + (T − I) equals exp(−iD/2) exp(−iΦJφ) exp(−iD/2) — catches the two misprints of Eq.
    lie_trotter_4 (reading R1) — and the diagonal keeps full relative precision near the identity."""
    rng = np.random.default_rng(3)
    for scale in (1.0, 1e-3, 1e-9):
        for _ in range(200):
            Phi, z, q = rng.uniform(0, scale), rng.uniform(-scale, scale), rng.uniform(-scale, scale)
            phi = rng.uniform(-np.pi, np.pi)
            D = z * J1Z + q * Q
            Jphi = np.cos(phi) * J1X + np.sin(phi) * J1Y
            a, b, c = _residual_series(D / 2), _residual_series(Phi * Jphi), _residual_series(D / 2)
            ref = a + b + c + a @ b + a @ c + b @ c + a @ b @ c           # (I+a)(I+b)(I+c) − I
            got = orc.trotter_residual(Phi, phi, z, q)
            # elementwise relative accuracy on the diagonal, absolute (scaled) elsewhere
            assert np.abs(got - ref).max() <= 1e-15 * scale
            if scale < 1:    # a "T − 1" implementation would lose ~|log10 scale| digits here
                for i in range(3):
                    assert abs(got[i, i] - ref[i, i]) <= 1e-14 * abs(ref[i, i]) + 1e-15 * scale
    # printed (uncorrected) T22 = cosΦ e^{i4q} would differ here:
    got = orc.trotter_residual(0.0, 0.0, 0.0, 0.3)
    assert abs(got[1, 1] - (np.exp(2j * 0.3 / 3) - 1)) < 1e-16


def test_lie_trotter_vs_expm_random(orc):
    """The paper's own exponentiator test: random matrices vs a general-purpose expm, τ = 24."""
    a = W.random_exponent_args(4000, 1.0, seed=4)
    U = orc.exponentiate("one", a, "lie_trotter", 24)
    ref = np.array([sl.expm(-1j * H_of("one", x)) for x in a])
    assert np.abs(U - ref).max() < 5e-15
    assert GOLD["trotter_cutoff_default"]["tau"] == 24


def test_lie_trotter_tau_sweep_monotone(orc):
    """Residual squaring: error falls ≈4^−τ (Strang) to the rounding floor with NO over-squaring rise
    (SURVEY [V2]; replaces SPEC's U-shape criterion, which holds only without residual squaring)."""
    a = W.random_exponent_args(300, 1.0, seed=5)
    ref = np.array([sl.expm(-1j * H_of("one", x)) for x in a])
    errs = [np.abs(orc.exponentiate("one", a, "lie_trotter", t) - ref).max() for t in range(0, 33, 4)]
    for e0, e1 in zip(errs[:5], errs[1:6]):               # τ = 0..20: each +4 squarings gains ≈ 4^4 = 256
        assert 60 < e0 / e1 < 1000
    assert max(errs[6:]) < 5e-15                          # τ ≥ 24 at the floor, no rise through τ = 32


def test_lie_trotter_structure(orc):
    # diagonal (commuting) case is exact: diag(e^{−i(θ+κ/3)}, e^{i2κ/3}, e^{−i(−θ+κ/3)})
    th, ka = 0.37, -1.3
    U = orc.exponentiate("one", [[0, 0, th, ka]], "lie_trotter", 24)[0]
    assert np.abs(U - np.diag(np.exp([-1j * (th + ka / 3), 2j * ka / 3, -1j * (-th + ka / 3)]))).max() < 1e-15
    a = W.random_exponent_args(200, 2.0, seed=6)
    Up = orc.exponentiate("one", a, "lie_trotter", 24)
    Um = orc.exponentiate("one", -a, "lie_trotter", 24)
    assert np.abs(Up @ Um - np.eye(3)).max() < 1e-14                         # inverse
    assert np.abs(np.conj(np.transpose(Up, (0, 2, 1))) @ Up - np.eye(3)).max() < 1e-14   # unitary
    assert np.abs(np.linalg.det(Up) - 1).max() < 1e-13


def test_spin_one_analytic_vs_expm(orc):
    a = W.random_exponent_args(2000, 1.5, seed=7, quad=False)
    U = orc.exponentiate("one", a, "analytic")
    ref = np.array([sl.expm(-1j * H_of("one", x)) for x in a])
    assert np.abs(U - ref).max() < 2e-15


def test_expm_dense_vs_scipy(orc):
    rng = np.random.default_rng(8)
    for d in (2, 3):
        for _ in range(50):
            X = rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))
            H = (X + X.conj().T) * 3
            assert np.abs(orc.expm_dense(H, 0.9) - sl.expm(-0.9j * H)).max() < 1e-13


# ---- fields and frame --------------------------------------------------------------------------------------
def test_field_examples(orc):
    g = GOLD["neural_pulse_parameters"]
    w, Om, Op = 2 * np.pi * g["omega_hz"], 2 * np.pi * g["Omega_hz"], 2 * np.pi * g["Omega_p_hz"]
    tp = 0.0233
    p = W.neural_params(w, w, Om, Op, Om, tp, 0.0)
    assert np.allclose(orc.field_sample("neural", p, 0.0, 0.0), [2 * Om, 0, w, 0], rtol=1e-15)
    t_peak = tp + (np.pi / 2) / Om
    f = orc.field_sample("neural", p, t_peak, 0.0)
    assert abs(f[2] - (w + Op)) < 1e-9 * w
    assert orc.field_sample("neural", p, tp + 1.5e-3, 0.0)[2] == w          # after the 1 ms pulse
    assert orc.field_sample("neural", p, tp - 1e-6, 0.0)[2] == w            # before it
    # sinp: one cycle only: pulse term is negative in the second half-cycle
    assert orc.field_sample("neural", p, tp + 0.75e-3, 0.0)[2] == pytest.approx(w - Op, rel=1e-12)
    # the (t_k, off) pair is the time t_k + off
    assert np.allclose(orc.field_sample("neural", p, 0.01, 3.3e-7), orc.field_sample("neural", p, 0.01 + 3.3e-7, 0.0),
                       rtol=1e-9)
    # Rabi examples
    w0, O = 2 * np.pi * 700e3, 2 * np.pi * 1e3
    assert np.allclose(orc.field_sample("rabi_linear", [w0, O], 0.0, 0.0), [2 * O, 0, w0, 0])
    assert np.allclose(orc.field_sample("rabi_linear", [w0, O], np.pi / w0, 0.0), [-2 * O, 0, w0, 0])
    assert np.allclose(orc.field_sample("rabi_circular", [w0, O], np.pi / (2 * w0), 0.0), [0, O, w0, 0], atol=1e-9)
    assert np.allclose(orc.field_sample("gradient", [3.0, 0.5], 1.0, 0.0), [0, 0, 2.0, 0])
    assert np.allclose(orc.field_sample("constant", [1, 2, 3, 4], 5.0, 0.0), [1, 2, 3, 4])


def test_rotating_frame_vs_conjugation(orc):
    """H_r = R(t)(ωxJx+ωyJy)R(−t) + (ωz−ω_r)Jz + ωqQ, R(t) = exp(iω_r Jz t), by explicit
    matrix conjugation, for both spins."""
    rng = np.random.default_rng(9)
    for _ in range(100):
        f = rng.standard_normal(4) * 1e3
        t, wr = rng.uniform(0, 1e-5), rng.uniform(-1e6, 1e6)
        g = orc.rotating_frame(f, t, wr)
        for spin in ("half", "one"):
            jx, jy, jz, q = ops(spin)
            R = sl.expm(1j * wr * jz * t)
            Hr = R @ (f[0] * jx + f[1] * jy) @ R.conj().T + (f[2] - wr) * jz + (f[3] * q if spin == "one" else 0)
            assert np.abs(H_of(spin, g if spin == "one" else np.r_[g[:3], 0]) - Hr).max() < 1e-9
        assert g[0] ** 2 + g[1] ** 2 == pytest.approx(f[0] ** 2 + f[1] ** 2, rel=1e-12)
    assert np.allclose(orc.rotating_frame([0, 0, 5.0, 0], 1e-3, 5.0), 0)         # frame nulling


# ---- [NS1] exact rotation under a constant field -----------------------------------------------------------
@pytest.mark.parametrize("spin,expo", [("half", "analytic"), ("one", "lie_trotter"), ("one", "analytic")])
def test_ns1_constant_field_frame_off_exact(orc, spin, expo):
    """Constant H: h1 = h2 = H/2 commute, so CF4 = exp(−iHδt) (Eq. exp_sol_of_constant) and
    U_k = exp(−iHΔt) exactly."""
    f = np.array([2.1e5, -1.3e5, 3.7e5, 0.0 if expo == "analytic" else 0.9e5])
    w = W.Workload("ns1", spin, "cf4", expo, 24, False, "constant", 0.0, 20e-6, 100e-9, 1e-6, f[None, :],
                   W.random_states(1, 2 if spin == "half" else 3, seed=10))
    st, U = run(orc, w)
    ref = sl.expm(-1j * H_of(spin, f) * 1e-6)
    assert np.abs(U[0] - ref).max() < 1e-13
    ts = np.arange(w.K + 1) * 1e-6
    exact = np.array([sl.expm(-1j * H_of(spin, f) * t) @ w.psi0[0] for t in ts])
    assert np.abs(st[0] - exact).max() < 1e-12


@pytest.mark.parametrize("spin", ["half", "one"])
def test_ns1_constant_bias_frame_on_nulls(orc, spin):
    """ωx = ωy = 0, frame on: ω_r = ωz nulls the in-frame field and U_k = exp(−iωz Jz Δt)."""
    wz = 2 * np.pi * 700e3
    w = W.Workload("ns1b", spin, "cf4", "lie_trotter" if spin == "one" else "analytic", 24, True, "constant",
                   0.0, 50e-6, 100e-9, 1e-6, np.array([[0.0, 0.0, wz, 0.0]]),
                   W.random_states(1, 2 if spin == "half" else 3, seed=11))
    st, U = run(orc, w)
    jz = ops(spin)[2]
    ref = np.diag(np.exp(-1j * wz * np.diag(jz).real * 1e-6))
    assert np.abs(U[0] - ref).max() < 1e-14
    ts = np.arange(w.K + 1) * 1e-6
    exact = np.array([np.exp(-1j * wz * np.diag(jz).real * t) * w.psi0[0] for t in ts])
    assert np.abs(st[0] - exact).max() < 1e-12


# ---- [NS2] Rabi formula ------------------------------------------------------------------------------------
def test_ns2_rabi_circular_resonant(orc):
    """Resonant circular drive, frame on (C1 grid): in-frame H is constant, so CF4 is exact and
    ψ(t) = e^{−iω0Jz t} e^{−iΩJx t} ψ0, P↓(t) = sin²(Ωt/2)."""
    w = W.c1_rabi("rabi_circular")
    st, _ = run(orc, w)
    w0, Om = w.sweep[0]
    ts = np.arange(w.K + 1) * w.dt_out
    P_down = np.abs(st[0][:, 1]) ** 2
    assert np.abs(P_down - np.sin(Om * ts / 2) ** 2).max() < 1e-12
    exact = np.array([sl.expm(-0.5j * w0 * t * SZ) @ sl.expm(-0.5j * Om * t * SX) @ [1, 0] for t in ts])
    assert np.abs(st[0] - exact).max() < 2e-12            # scipy's own phase rounding at ω0 t ≈ 4.4e3 rad


def test_ns2_rabi_linear_drive_rwa(orc):
    """The paper-form linear drive 2Ω cos(ω0 t) Jx agrees with the Rabi formula only to the RWA."""
    w = W.c1_rabi("rabi_linear")
    st, _ = run(orc, w)
    Om = w.sweep[0, 1]
    ts = np.arange(w.K + 1) * w.dt_out
    assert np.abs(np.abs(st[0][:, 1]) ** 2 - np.sin(Om * ts / 2) ** 2).max() < 1e-3


# ---- [NS3] spin-one = symmetric (spin-1) representation of spin-half when ωq = 0 --------------------------
@pytest.mark.parametrize("expo", ["lie_trotter", "analytic"])
def test_ns3_spin_one_is_symmetric_rep(orc, expo):
    p = W.neural_params(t_p=0.2e-3, omega_q=0.0)
    half = W.Workload("h", "half", "cf4", "analytic", 24, True, "neural", 0.0, 0.5e-3, 100e-9, 1e-6, p[None, :],
                      W.random_states(1, 2, seed=12))
    a0, b0 = half.psi0[0]
    one = half.with_(spin="one", expo=expo, psi0=np.array([[a0 * a0, math.sqrt(2) * a0 * b0, b0 * b0]]))
    sh, _ = run(orc, half)
    s1, _ = run(orc, one)
    al, be = sh[0][:, 0], sh[0][:, 1]
    sym = np.stack([al * al, math.sqrt(2) * al * be, be * be], axis=1)
    assert np.abs(s1[0] - sym).max() < 1e-12


# ---- [NS4] unitarity ---------------------------------------------------------------------------------------
@pytest.mark.parametrize("spin,expo", [("half", "analytic"), ("one", "lie_trotter")])
def test_ns4_unitarity(orc, spin, expo):
    w = W.c2_neural(duration=2e-3).with_(spin=spin, expo=expo, psi0=W.random_states(1, 2 if spin == "half" else 3, 13))
    st, U = run(orc, w)
    d = w.dim
    UhU = np.conj(np.transpose(U[0], (0, 2, 1))) @ U[0]
    assert np.abs(UhU - np.eye(d)).max() < 1e-12           # every interval operator
    assert np.abs(np.linalg.norm(st[0], axis=1) - 1).max() < 1e-12     # K = 2e3 ≪ 3e4


# ---- [NS5] 4th-order convergence of CF4 (and 2nd order of the Euler samplers) -----------------------------
def _dop853_reference(spin, field_fn, t_end, psi0, n_out):
    def rhs(t, y):
        psi = y[: len(y) // 2] + 1j * y[len(y) // 2:]
        d = -1j * (H_of(spin, field_fn(t)) @ psi)
        return np.r_[d.real, d.imag]
    ts = np.linspace(0, t_end, n_out)
    sol = si.solve_ivp(rhs, (0, t_end), np.r_[psi0.real, psi0.imag], method="DOP853", t_eval=ts,
                       rtol=1e-13, atol=1e-13, max_step=2e-8)
    y = sol.y.T
    return y[:, : len(psi0)] + 1j * y[:, len(psi0):]


def _neural_field_fn(p):
    """Eq. neural_pulse written out in the test (the problem statement, not the method)."""
    wb, wrf, Om, Op, ws, tp, wq = p
    def f(t):
        x = ws * (t - tp)
        pulse = math.sin(x) if 0 <= x <= 2 * math.pi else 0.0
        return np.array([2 * Om * math.cos(wrf * t), 0.0, wb + Op * pulse, wq])
    return f


@pytest.mark.parametrize("spin,expo,frame", [("half", "analytic", True), ("half", "analytic", False),
                                             ("one", "lie_trotter", True)])
def test_ns5_cf4_fourth_order(orc, spin, expo, frame):
    # Strong dressing so the truncation error sits well above the rounding floor on a short window.
    p = W.neural_params(omega_bias=2 * np.pi * 200e3, omega_dress=2 * np.pi * 40e3, omega_sig=2 * np.pi * 100e3,
                        omega_pulse=2 * np.pi * 20e3, t_p=5e-6, omega_q=2 * np.pi * 3e3 if spin == "one" else 0.0)
    t_end, dt_out = 20e-6, 2e-6
    d = 2 if spin == "half" else 3
    psi0 = W.random_states(1, d, seed=14)
    ref = _dop853_reference(spin, _neural_field_fn(p), t_end, psi0[0], int(round(t_end / dt_out)) + 1)
    errs = {}
    for method in ("cf4", "midpoint"):
        errs[method] = []
        for dt in (500e-9, 250e-9, 125e-9, 62.5e-9):
            w = W.Workload("ns5", spin, method, expo, 24, frame, "neural", 0.0, t_end, dt, dt_out, p[None, :], psi0)
            st, _ = run(orc, w, want_unitaries=False)
            errs[method].append(np.abs(st[0] - ref).max())
    r4 = [a / b for a, b in zip(errs["cf4"], errs["cf4"][1:])]
    r2 = [a / b for a, b in zip(errs["midpoint"], errs["midpoint"][1:])]
    assert all(10 <= r <= 24 for r in r4), (errs["cf4"], r4)
    assert all(3 <= r <= 6 for r in r2), (errs["midpoint"], r2)
    assert errs["cf4"][-1] > 1e-11                          # still above the reference's floor


def test_heun_second_order_and_constant_exact(orc):
    f = np.array([1.1e5, 0.4e5, -2e5, 0.0])
    w = W.Workload("h", "half", "heun", "analytic", 24, False, "constant", 0.0, 5e-6, 100e-9, 1e-6, f[None, :],
                   W.basis_state(2))
    _, U = run(orc, w)
    assert np.abs(U[0] - sl.expm(-1j * H_of("half", f) * 1e-6)).max() < 1e-14
    p = W.neural_params(omega_bias=2 * np.pi * 200e3, omega_dress=2 * np.pi * 40e3, omega_sig=2 * np.pi * 100e3,
                        omega_pulse=2 * np.pi * 20e3, t_p=5e-6, omega_q=0.0)
    psi0 = W.random_states(1, 2, seed=15)
    ref = _dop853_reference("half", _neural_field_fn(p), 20e-6, psi0[0], 11)
    errs = []
    for dt in (250e-9, 125e-9, 62.5e-9):
        w = W.Workload("h", "half", "heun", "analytic", 24, True, "neural", 0.0, 20e-6, dt, 2e-6, p[None, :], psi0)
        errs.append(np.abs(run(orc, w, want_unitaries=False)[0][0] - ref).max())
    assert all(3 <= a / b <= 6 for a, b in zip(errs, errs[1:])), errs


# ---- chain, projection, error metric ----------------------------------------------------------------------
def test_chain_accumulate_example(orc):
    """−iσx applied to (1,0) → (0,−i): constant ωx = π/Δt over one interval, frame off."""
    w = W.Workload("acc", "half", "cf4", "analytic", 24, False, "constant", 0.0, 1e-6, 1e-6, 1e-6,
                   np.array([[np.pi / 1e-6, 0, 0, 0]]), W.basis_state(2))
    st, _ = run(orc, w)
    g = np.array(GOLD["accumulate_example"]["psi_out"], float)
    assert np.abs(st[0][1] - (g[:, 0] + 1j * g[:, 1])).max() < 1e-15


def test_chain_matches_product_of_unitaries(orc):
    w = W.c2_neural(duration=0.2e-3).with_(psi0=W.random_states(1, 3, seed=16))
    st, U = run(orc, w)
    psi = w.psi0[0].copy()
    for k in range(w.K):
        psi = U[0][k] @ psi
        assert np.abs(st[0][k + 1] - psi).max() < 1e-14


def test_spin_projection_examples(orc):
    for case in GOLD["spin_projection_examples"]["cases"]:
        psi = np.array(case["psi"], float)
        got = orc.spin_projection(case["spin"], (psi[:, 0] + 1j * psi[:, 1])[None, :])[0]
        assert np.allclose(got, case["J"], atol=1e-15)
    rng = np.random.default_rng(17)
    for spin in ("half", "one"):
        d = 2 if spin == "half" else 3
        psi = W.random_states(20, d, seed=18)
        got = orc.spin_projection(spin, psi)
        jx, jy, jz, _ = ops(spin)
        ref = np.stack([np.einsum("ni,ij,nj->n", psi.conj(), j, psi).real for j in (jx, jy, jz)], axis=1)
        assert np.abs(got - ref).max() < 1e-15
    del rng


def test_rms_error_examples(orc):
    a = np.array([[1, 0]], complex)
    b = np.array([[0, 1]], complex)
    assert orc.rms_error(a, b) == pytest.approx(GOLD["rms_error_examples"]["K1_orthogonal"], rel=1e-15)
    assert orc.rms_error(np.repeat(a, 4, 0), np.repeat(b, 4, 0)) == pytest.approx(
        GOLD["rms_error_examples"]["K4_orthogonal"], rel=1e-15)
    assert orc.rms_error(a, a) == 0


def test_double_and_long_double_instantiations_agree(orc):
    w = W.c2_neural(duration=1e-3)
    a, _ = run(orc, w, want_unitaries=False)
    b, _ = run(orc, w, want_unitaries=False, long_double=False)
    assert np.abs(a - b).max() < 1e-11


def test_frame_on_off_converge(orc):
    """Frame on and off solve the same problem: their difference shrinks as δt → 0."""
    p = W.neural_params(t_p=0.0, omega_q=W.OMEGA_Q)
    diffs = []
    for dt in (50e-9, 25e-9):
        w = W.Workload("f", "one", "cf4", "lie_trotter", 24, True, "neural", 0.0, 10e-6, dt, 1e-6, p[None, :],
                       W.basis_state(3))
        on, _ = run(orc, w, want_unitaries=False)
        off, _ = run(orc, w.with_(frame=False), want_unitaries=False)
        diffs.append(np.abs(on - off).max())
    assert diffs[1] < diffs[0] / 8


def test_k_range_subset_matches_full(orc):
    w = W.c3_batched(batch=3, duration=50e-6)
    full_st, full_U = run(orc, w)
    st, U = run(orc, w, k_begin=20, k_end=30)
    assert np.array_equal(U, full_U[:, 20:30])


@pytest.mark.parametrize("spin,expo", [("half", "analytic"), ("one", "lie_trotter")])
def test_interval_operator_composition(orc, spin, expo):
    """U_k = R_{ω_r}(−Δt) u_{L−1}⋯u_0 with ω_r = ω_z(t_k + Δt/2) sampled from the lab field,
    rebuilt here from single fine steps with the paper's ω_r rule and exit factor exp(−iω_r Jz Δt)."""
    w = W.c2_neural(dt_int=250e-9, duration=40e-6).with_(spin=spin, expo=expo, psi0=W.basis_state(2 if spin == "half" else 3),
                                                           sweep=W.neural_params(t_p=5e-6)[None, :])
    p = w.sweep[0]                      # pulse active inside the window, so ω_z varies within intervals
    _, U = run(orc, w)
    jz = np.diag(ops(spin)[2]).real
    for k in (0, 17, 39):
        t_k = orc.grid(w.t0, w.dt_out, w.dt_int, k, 0)["t_k"]
        wr = orc.field_sample("neural", p, t_k, 0.5 * w.dt_out)[2]
        acc = np.eye(w.dim, dtype=complex)
        for l in range(w.L):
            acc = orc.fine_step(spin, "cf4", expo, 24, True, "neural", p, w.t0, w.dt_out, w.dt_int, k, l, wr) @ acc
        ref = np.diag(np.exp(-1j * wr * jz * w.dt_out)) @ acc
        assert np.abs(U[0][k] - ref).max() < 1e-15
