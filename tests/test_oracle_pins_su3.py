"""Pins for the oracle's general spin-one (su(3)) exponentiator and fields (P:184-189,
P:478-479; readings R19, R20).  Every check ties the oracle to something other than itself: the operator
matrices are built HERE from the textbook spin-1 matrices (U1 = Jx² − Jy², U2 = {Jx, Jy}, V1 = {Jx, Jz},
V2 = {Jy, Jz}), exponentials come from scipy.linalg.expm / mpmath, the full path from a closed-form lab solution
and from scipy's DOP853.  These run without a GPU.
"""
import math

import mpmath
import numpy as np
import pytest
import scipy.integrate as si
import scipy.linalg as sl

import workloads as W

R2 = 1 / math.sqrt(2)
JX = R2 * np.array([[0, 1, 0], [1, 0, 1], [0, 1, 0]], complex)
JY = R2 * np.array([[0, -1j, 0], [1j, 0, -1j], [0, 1j, 0]], complex)
JZ = np.diag([1.0, 0.0, -1.0]).astype(complex)
Q = np.diag([1.0, -2.0, 1.0]).astype(complex) / 3
U1 = JX @ JX - JY @ JY                                          # Δm = ±2 quadrupoles (reading R19)
U2 = JX @ JY + JY @ JX
V1 = JX @ JZ + JZ @ JX                                          # Δm = ±1 quadrupoles
V2 = JY @ JZ + JZ @ JY
BASIS = [JX, JY, JZ, Q, U1, U2, V1, V2]


def H8(a):
    return sum(x * A for x, A in zip(a, BASIS))


def run(orc, w, **kw):
    return orc.evaluate(w.spin, w.method, w.expo, w.tau, w.frame, w.field, sweep=w.sweep, t0=w.t0, t1=w.t1,
                        dt_int=w.dt_int, dt_out=w.dt_out, psi0=w.psi0, **kw)


def test_basis_spans_su3():
    """The 8 operators are traceless, Hermitian and linearly independent (they span su(3))."""
    G = np.array([[np.trace(A @ B).real for B in BASIS] for A in BASIS])
    assert abs(np.linalg.det(G)) > 1e-3
    for A in BASIS:
        assert abs(np.trace(A)) < 1e-15 and np.abs(A - A.conj().T).max() < 1e-15
    # Δm structure used by the frame rotation: U couples m = ±1 only, V and J couple Δm = ±1
    assert np.abs(U1 - np.array([[0, 0, 1], [0, 0, 0], [1, 0, 0]])).max() < 1e-15
    assert np.abs(np.diag(np.diag(V1)) ).max() == 0


def test_single_operators_vs_expm(orc):
    """Each basis operator alone: the oracle maps coefficient j to operator j (catches a swapped or mis-signed
    operator in the exponentiator's matrix assembly)."""
    for j in range(8):
        for x in (0.3, -1.1, 2.5):
            a = np.zeros(8)
            a[j] = x
            got = orc.exponentiate("one", a[None, :], "lie_trotter_su3", 24)[0]
            assert np.abs(got - sl.expm(-1j * x * BASIS[j])).max() < 5e-15, (j, x)


def test_su3_lie_trotter_vs_expm_random(orc):
    """The paper's exponentiator test extended to all 8 coefficients, τ = 24."""
    a = W.random_exponent_args_su3(3000, 1.0, seed=21)
    U = orc.exponentiate("one", a, "lie_trotter_su3", 24)
    ref = np.array([sl.expm(-1j * H8(x)) for x in a])
    assert np.abs(U - ref).max() < 1e-14


def test_su3_four_operator_case(orc):
    """With au = av = 0 the basis product (reading R20) and the paper's own factor of Eq. lie_trotter_4 are two
    second-order splittings of the same exponential: both within rounding of expm at τ = 24, so they agree there; at
    τ = 0 they are different splittings (the paper groups Jx, Jy into one rotation ΦJφ)."""
    a4 = W.random_exponent_args(300, 1.0, seed=22)
    a8 = np.concatenate([a4, np.zeros((300, 4))], axis=1)
    d = np.abs(orc.exponentiate("one", a8, "lie_trotter_su3", 24) - orc.exponentiate("one", a4, "lie_trotter", 24))
    assert d.max() < 5e-15
    d0 = np.abs(orc.exponentiate("one", a8, "lie_trotter_su3", 0) - orc.exponentiate("one", a4, "lie_trotter", 0))
    assert d0.max() > 1e-3


def test_su3_tau_sweep(orc):
    """Strang splitting: error vs expm falls ≈ 4^−τ to the rounding floor, no over-squaring rise (reading R17)."""
    a = W.random_exponent_args_su3(200, 1.0, seed=23)
    ref = np.array([sl.expm(-1j * H8(x)) for x in a])
    errs = [np.abs(orc.exponentiate("one", a, "lie_trotter_su3", t) - ref).max() for t in range(0, 33, 4)]
    for e0, e1 in zip(errs[:5], errs[1:6]):
        assert 60 < e0 / e1 < 1000, errs
    assert max(errs[6:]) < 1e-14, errs


# Leapfrog order of the basis product (reading R20): diagonal operators (Jz, Q) outermost as in P:374, then U1, U2,
# V1, V2, Jx, and Jy in the middle with the full step.
OUTER, MIDDLE = (2, 3, 4, 5, 6, 7, 0), 1


def _mp_basis_product_residual(a, n):
    """T − I of the leapfrog basis product in 40-digit arithmetic: mpmath.expm of each single operator −i·frac·a_j·A_j/n
    (the test's own matrices), multiplied out in order, then I subtracted (no cancellation at this precision)."""
    with mpmath.workdps(40):
        def ex(j, frac):
            M = mpmath.matrix([[mpmath.mpc(complex(BASIS[j][r, c])) for c in range(3)] for r in range(3)])
            return mpmath.expm(M * (-1j) * mpmath.mpf(a[j]) * frac / n)
        T = mpmath.eye(3)
        for j in OUTER:
            T = T * ex(j, mpmath.mpf(1) / 2)
        T = T * ex(MIDDLE, 1)
        for j in reversed(OUTER):
            T = T * ex(j, mpmath.mpf(1) / 2)
        T = T - mpmath.eye(3)
        return np.array([[complex(T[i, j]) for j in range(3)] for i in range(3)])


def test_su3_factor_residual_vs_mpmath(orc):
    """T − I of the basis product (reading R20) against 40-digit arithmetic — elementwise RELATIVE accuracy
    (the residual form keeps the digits P:463-466 asks for, which subtracting I from T would lose), at a large and a
    tiny argument scale."""
    rng = np.random.default_rng(24)
    for scale, tau in ((1.0, 0), (1.0, 20), (1e-4, 24)):
        for _ in range(6):
            a = rng.uniform(-scale, scale, 8)
            ref = _mp_basis_product_residual(a, 2.0 ** tau)
            got = orc.trotter_residual_su3(a, tau)
            assert np.all(np.abs(got - ref) <= 1e-15 * np.abs(ref) + 1e-16 * scale / 2.0 ** tau), (scale, tau, got - ref)


def test_su3_factor_properties(orc):
    """Properties of the factor that do not depend on the splitting order: (i) unitary for any argument, (ii) exact
    when only the commuting diagonal operators (Jz, Q) are present, (iii) T = exp(−iH/n) + O(|H/n|³) — a symmetric
    (second-order) splitting: halving the argument divides the error by ≈ 8 (a first-order product would give ≈ 4)."""
    rng = np.random.default_rng(25)
    for _ in range(50):
        a = rng.uniform(-2, 2, 8)
        T = orc.trotter_residual_su3(a, 0) + np.eye(3)
        assert np.abs(T.conj().T @ T - np.eye(3)).max() < 1e-15
    a = np.array([0, 0, 0.7, -1.9, 0, 0, 0, 0])
    assert np.abs(orc.trotter_residual_su3(a, 0) + np.eye(3) - sl.expm(-1j * H8(a))).max() < 1e-16
    for a in (np.array([0.4, 0.4, 0.3, -0.7, 0, 0, -0.4, -0.4]), np.array([0, 0, 0.2, 0.1, 0.8, -0.6, 0, 0]),
              rng.uniform(-1, 1, 8)):
        errs = []
        for s in (0.2, 0.1, 0.05):
            T = orc.trotter_residual_su3(s * a, 0) + np.eye(3)
            errs.append(np.abs(T - sl.expm(-1j * H8(s * a))).max())
        assert 6.5 < errs[0] / errs[1] < 9.5 and 6.5 < errs[1] / errs[2] < 9.5, errs


def test_su3_basis_closed_forms():
    """The closed form the oracle uses for the non-diagonal factors needs A³ = A (eigenvalues 0, ±1) for Jx, Jy, U1,
    U2, V1, V2; Jz and Q are diagonal."""
    for j in (0, 1, 4, 5, 6, 7):
        A = BASIS[j]
        assert np.abs(A @ A @ A - A).max() < 1e-15, j
        th = 0.37
        E = np.eye(3) - 1j * np.sin(th) * A + (np.cos(th) - 1) * (A @ A)
        assert np.abs(E - sl.expm(-1j * th * A)).max() < 1e-15, j
    for j in (2, 3):
        assert np.abs(BASIS[j] - np.diag(np.diag(BASIS[j]))).max() == 0


def test_su3_structure(orc):
    a = W.random_exponent_args_su3(200, 2.0, seed=25)
    Up = orc.exponentiate("one", a, "lie_trotter_su3", 24)
    Um = orc.exponentiate("one", -a, "lie_trotter_su3", 24)
    assert np.abs(Up @ Um - np.eye(3)).max() < 1e-14
    assert np.abs(np.conj(np.transpose(Up, (0, 2, 1))) @ Up - np.eye(3)).max() < 1e-14   # unitary
    assert np.abs(np.linalg.det(Up) - 1).max() < 1e-13                                   # SU(3)
    # diagonal case exact
    U = orc.exponentiate("one", np.array([[0, 0, 0.37, -1.3, 0, 0, 0, 0]]), "lie_trotter_su3", 24)[0]
    assert np.abs(U - sl.expm(-1j * (0.37 * JZ - 1.3 * Q))).max() < 1e-15


def test_su3_expo_rejected_for_spin_half_and_su3_fields_need_it(orc):
    with pytest.raises(ValueError):
        orc.exponentiate("half", np.zeros((1, 8)), "lie_trotter_su3")
    w = W.g1_su3(batch=1, duration=2e-6)
    with pytest.raises(ValueError):
        run(orc, w.with_(expo="lie_trotter"))


def test_su3_field_examples(orc):
    w0, wq, Ox, Ov, Ou, wd = W.su3_drive_params(omega_d=2 * np.pi * 650e3)
    p = W.su3_drive_params(omega_d=2 * np.pi * 650e3)
    assert np.allclose(orc.field_sample("su3_drive", p, 0.0, 0.0), [Ox, 0, w0, wq, Ou, 0, Ov, 0], rtol=1e-15)
    t = np.pi / (2 * wd)                          # quarter period: (cos, sin) = (0, 1); two-photon at half period
    assert np.allclose(orc.field_sample("su3_drive", p, t, 0.0), [0, Ox, w0, wq, -Ou, 0, 0, Ov], atol=1e-9 * w0)
    assert np.allclose(orc.field_sample("su3_constant", np.arange(1, 9), 3.0, 0.0), np.arange(1, 9))


def test_su3_rotating_frame_vs_conjugation(orc):
    """H_r = R H R† − ω_r Jz with R = exp(iω_r Jz t) by explicit conjugation, all 8 coefficients."""
    rng = np.random.default_rng(26)
    for _ in range(100):
        f = rng.standard_normal(8) * 1e3
        t, wr = rng.uniform(0, 1e-5), rng.uniform(-1e6, 1e6)
        g = orc.rotating_frame(f, t, wr)
        R = sl.expm(1j * wr * JZ * t)
        Hr = R @ H8(f) @ R.conj().T - wr * JZ
        assert np.abs(H8(g) - Hr).max() < 1e-9


def test_su3_constant_field_frame_off_exact(orc):
    """Constant H: CF4 is exp(−iHδt) and U_k = exp(−iHΔt) (Eq. exp_sol_of_constant)."""
    f = np.array([2.1e5, -1.3e5, 3.7e5, 0.9e5, -1.7e5, 0.6e5, 1.2e5, -2.2e5])
    w = W.Workload("su3c", "one", "cf4", "lie_trotter_su3", 24, False, "su3_constant", 0.0, 20e-6, 100e-9, 1e-6,
                   f[None, :], W.random_states(1, 3, seed=27))
    st, U = run(orc, w)
    assert np.abs(U[0] - sl.expm(-1j * H8(f) * 1e-6)).max() < 1e-13
    exact = np.array([sl.expm(-1j * H8(f) * t) @ w.psi0[0] for t in np.arange(w.K + 1) * 1e-6])
    assert np.abs(st[0] - exact).max() < 1e-12


def test_su3_drive_resonant_closed_form(orc):
    """Resonant drive (ω_d = ω0), frame on: H(t) = e^{−iω0Jz t} H' e^{iω0Jz t} + ω0 Jz with the constant
    H' = ω_q Q + Ω_x Jx + Ω_v V1 + Ω_u U1, so ψ(t) = e^{−iω0 Jz t} e^{−iH' t} ψ0 exactly; in the frame the field is
    constant per interval and CF4 is exact.  Exercises every operator, the U-pair 2θ frame rotation and the exit."""
    p = W.su3_drive_params(omega_x=2 * np.pi * 3e3, omega_v=2 * np.pi * 1.3e3, omega_u=2 * np.pi * 2e3)
    w = W.Workload("su3r", "one", "cf4", "lie_trotter_su3", 24, True, "su3_drive", 0.0, 1e-3, 100e-9, 1e-6,
                   p[None, :], W.random_states(1, 3, seed=28))
    st, _ = run(orc, w, want_unitaries=False)
    w0, wq, Ox, Ov, Ou, _ = p
    Hp = wq * Q + Ox * JX + Ov * V1 + Ou * U1
    ts = np.arange(w.K + 1) * w.dt_out
    exact = np.array([np.exp(-1j * w0 * np.diag(JZ).real * t) * (sl.expm(-1j * Hp * t) @ w.psi0[0]) for t in ts])
    assert np.abs(st[0] - exact).max() < 3e-12            # phase rounding at ω0 t ≈ 4.4e3 rad, as in [NS2]
    # populations move between all three levels (the drive is not trivial)
    assert np.abs(st[0][:, 1]).max() > 0.3


def test_su3_drive_detuned_fourth_order(orc):
    """Detuned drive (in-frame field rotates): CF4 error vs DOP853 on the lab H falls ×16 per δt halving."""
    p = W.su3_drive_params(omega0=2 * np.pi * 200e3, omega_q=2 * np.pi * 5e3, omega_x=2 * np.pi * 30e3,
                           omega_v=2 * np.pi * 12e3, omega_u=2 * np.pi * 9e3, omega_d=2 * np.pi * 180e3)
    w0, wq, Ox, Ov, Ou, wd = p

    def rhs(t, y):
        c, s, c2, s2 = math.cos(wd * t), math.sin(wd * t), math.cos(2 * wd * t), math.sin(2 * wd * t)
        H = H8([Ox * c, Ox * s, w0, wq, Ou * c2, Ou * s2, Ov * c, Ov * s])
        psi = y[:3] + 1j * y[3:]
        d = -1j * (H @ psi)
        return np.r_[d.real, d.imag]

    psi0 = W.random_states(1, 3, seed=29)
    t_end, dt_out = 20e-6, 2e-6
    ts = np.linspace(0, t_end, 11)
    sol = si.solve_ivp(rhs, (0, t_end), np.r_[psi0[0].real, psi0[0].imag], method="DOP853", t_eval=ts,
                       rtol=1e-13, atol=1e-13, max_step=2e-8)
    ref = (sol.y[:3] + 1j * sol.y[3:]).T
    errs = []
    for dt in (500e-9, 250e-9, 125e-9, 62.5e-9):
        w = W.Workload("su3d", "one", "cf4", "lie_trotter_su3", 24, True, "su3_drive", 0.0, t_end, dt, dt_out,
                       p[None, :], psi0)
        errs.append(np.abs(run(orc, w, want_unitaries=False)[0][0] - ref).max())
    r = [a / b for a, b in zip(errs, errs[1:])]
    assert all(10 <= x <= 24 for x in r), (errs, r)
    assert errs[-1] > 1e-11


# ---- Magnus-convergence diagnostic ------------------------------------------------------------
def test_spectral_norm_vs_eigvalsh(orc):
    """‖H‖₂ of the oracle's dense Hamiltonian (assembled from the operator definitions) = max |eigvalsh| of the
    test's own H8 (spin-one) / σ/2 (spin-half), over random coefficients."""
    rng = np.random.default_rng(51)
    for _ in range(300):
        f = rng.standard_normal(8) * rng.choice([1e-3, 1.0, 1e4])
        ref = np.abs(np.linalg.eigvalsh(H8(f))).max()
        assert abs(orc.spectral_norm("one", f) - ref) <= 1e-12 * ref
        h2 = 0.5 * (f[0] * np.array([[0, 1], [1, 0]]) + f[1] * np.array([[0, -1j], [1j, 0]])
                    + f[2] * np.diag([1.0, -1.0]))
        ref2 = np.abs(np.linalg.eigvalsh(h2)).max()
        assert abs(orc.spectral_norm("half", f[:3]) - ref2) <= 1e-12 * ref2


def test_magnus_bound_spec_examples(orc):
    """S:161-169 examples: field-norm bound × δt against ξ = 1.08686870.  Constant spin-half field with
    ‖H‖₂ = |ω|/2 = 2π·1e6 rad/s, frame off: 0.628 at δt = 100 ns (converges), 1.257 at 200 ns (does not)."""
    w = 2 * 2 * np.pi * 1e6
    for dt, conv in ((1e-7, True), (2e-7, False)):
        mb = orc.magnus_bound("half", False, "constant", sweep=[[w, 0, 0, 0]], t0=0.0, t1=4e-6, dt_int=dt,
                              dt_out=4e-7)[0]
        assert mb == pytest.approx(np.pi * 2e6 * dt, rel=1e-15)
        assert (mb < orc.MAGNUS_XI) == conv
    # the frame removes the bias: a pure z field has zero in-frame norm; the quadratic shift keeps 2|ωq|/3
    mb = orc.magnus_bound("one", True, "constant", sweep=[[0, 0, 4.4e6, 3e3]], t0=0.0, t1=2e-6, dt_int=1e-7,
                          dt_out=1e-6)[0]
    assert mb == pytest.approx(2 / 3 * 3e3 * 1e-7, rel=1e-12)


def test_magnus_bound_is_max_gauss_estimate(orc):
    """Brute force: the diagnostic equals the maximum over steps of the Gauss–Legendre estimate rebuilt here from the
    oracle's field samples, frame rotation and numpy eigenvalues."""
    w = W.g1_su3(batch=2, duration=4e-6)
    p = w.sweep[1]
    g1, g2 = orc.constants()["g1"], orc.constants()["g2"]
    dt = w.dt_int
    worst = 0.0
    for k in range(w.K):
        t_k = k * w.dt_out
        wr = orc.field_sample("su3_drive", p, t_k, 0.5 * w.dt_out)[2]
        for l in range(w.L):
            n = []
            for g in (g1, g2):
                off = l * dt + g * dt
                f = orc.rotating_frame(orc.field_sample("su3_drive", p, t_k, off), off, wr)
                n.append(np.abs(np.linalg.eigvalsh(H8(f))).max())
            worst = max(worst, dt * (n[0] + n[1]) / 2)
    got = orc.magnus_bound("one", True, "su3_drive", sweep=w.sweep, t0=w.t0, t1=w.t1, dt_int=w.dt_int,
                           dt_out=w.dt_out)[1]
    assert got == pytest.approx(worst, rel=1e-9)
