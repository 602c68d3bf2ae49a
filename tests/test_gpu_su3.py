"""GPU parity of the general spin-one (su(3)) path (readings R19, R20):
the CUDA kernels through the C ABI against the long-double oracle on the same seeded inputs, element by element.
Bars as everywhere: 1e-10 (FP64), 1e-4 (FP32 mode, rotating frame on)."""
import numpy as np
import pytest
import torch

import workloads as W

pytestmark = pytest.mark.gpu

TOL64 = 1e-10
TOL32 = 1e-4


def splitting_tol(scale, tau):
    """The GPU's tridiagonalised factor and the oracle's basis product are different second-order (Strang)
    splittings (reading R20): each is exp(−iH) + O(|a|³/n²), n = 2^τ, so exponentials of |a| ≲ √8·scale differ by up
    to ≈ (√8·scale)³·4^−τ/3 on top of rounding."""
    return (np.sqrt(8) * scale) ** 3 * 4.0 ** -tau / 3


@pytest.fixture(scope="module")
def ss():
    import paper_2204_05586_b200 as ss
    assert torch.cuda.is_available()
    ss.load()
    return ss


def parity(ss, orc, w, precision="fp64", tol=TOL64):
    sim = ss.Simulator(w.spin, w.method, w.expo, w.tau, w.frame, precision, w.field)
    res = sim.evaluate(torch.from_numpy(np.ascontiguousarray(w.sweep)).cuda(), w.t0, w.t1, w.dt_int, w.dt_out,
                       torch.from_numpy(np.ascontiguousarray(w.psi0)).cuda())
    torch.cuda.synchronize()
    st_o, U_o = orc.evaluate(w.spin, w.method, w.expo, w.tau, w.frame, w.field, sweep=w.sweep, t0=w.t0, t1=w.t1,
                             dt_int=w.dt_int, dt_out=w.dt_out, psi0=w.psi0)
    eU = np.abs(res.time_evolution.cpu().numpy() - U_o).max()
    eS = np.abs(res.state.cpu().numpy() - st_o).max()
    assert eU <= tol and eS <= tol, (w.name, precision, eU, eS)
    return eU, eS


@pytest.mark.parametrize("scale", [2.0, 0.03, 0.025, 0.01, 1e-3, 1e-7])   # 0.03 / 0.025 straddle the Taylor bound
def test_su3_exponentiator_parity(ss, orc, scale):
    a = W.random_exponent_args_su3(5000, scale, seed=31)
    a[:2] = 0.0                                   # exact zero (identity)
    a[2, [0, 1, 4, 5, 6, 7]] = 0.0                # diagonal only
    a[3, [4, 5]] = 0.0                            # no (0,2) coupling
    a[4, [0, 1, 6, 7]] = 0.0                      # (0,2) coupling only
    a[5, [4, 5]] = 0.0                            # H01 = H02 = 0 (r = 0: W is the phase alone, reading R20)
    a[5, [6, 7]] = -a[5, [0, 1]]
    a[6, [6, 7]] = a[6, [0, 1]]                   # H12 = 0
    a[7, [6, 7]] = a[7, [0, 1]]                   # H12 = 0 and H02 = 0: B12 = 0 (no phase)
    a[7, [4, 5]] = 0.0
    tau = 24 if scale < 1 else 30               # large arguments: τ = 30 keeps the splitting difference below rounding
    ref = orc.exponentiate("one", a, "lie_trotter_su3", tau)
    for prec, tol in (("fp64", 4e-15 * max(1.0, scale) + splitting_tol(scale, tau)), ("fp32", 2e-6)):
        sim = ss.Simulator("one", "cf4", "lie_trotter_su3", tau, True, prec, "su3_constant")
        got = sim.exponentiate(torch.from_numpy(a).cuda()).cpu().numpy()
        assert np.abs(got - ref).max() <= tol, (prec, np.abs(got - ref).max())


def test_su3_tiny_couplings(ss, orc):
    """Couplings down to 1e-30 next to O(1) diagonals (FP32 subnormal range for |H01|², |H02|²): the similarity W of
    reading R20 stays finite and unitary, so the exponential is the diagonal one plus the tiny coupling."""
    a = np.zeros((6, 8))
    a[:, 2], a[:, 3] = 0.7, -0.4
    a[0, [0, 1]] = [1e-30, -2e-30]                 # H01 = H12 tiny
    a[1, [4, 5]] = [3e-21, 1e-21]                  # H02 tiny
    a[2, [0, 6]] = [1e-19, 1e-19]                  # H01 tiny-ish, H12 = 0
    a[3, [0, 6]] = [0.3, -0.3 + 1e-18]             # H01 ≈ 1e-18, H12 ≈ 0.42
    a[4, :] = 0.0
    a[4, 4] = 1e-300                               # FP64 only: H02 at the bottom of the double range
    a[5, [0, 4, 7]] = [1e-25, 0.2, 1e-25]
    ref = orc.exponentiate("one", a, "lie_trotter_su3", 24)
    for prec, tol in (("fp64", 4e-15 + splitting_tol(0.7, 24)), ("fp32", 2e-6)):
        sim = ss.Simulator("one", "cf4", "lie_trotter_su3", 24, True, prec, "su3_constant")
        got = sim.exponentiate(torch.from_numpy(a).cuda()).cpu().numpy()
        assert np.isfinite(got).all(), prec
        assert np.abs(got - ref).max() <= tol, (prec, np.abs(got - ref).max(axis=(1, 2)))


@pytest.mark.parametrize("tau", [24, 33])
def test_su3_tau_parity(ss, orc, tau):
    """At τ ≥ 20 both splittings are within rounding of exp(−iH): GPU vs the oracle's basis product."""
    a = W.random_exponent_args_su3(500, 0.5, seed=32)
    sim = ss.Simulator("one", "cf4", "lie_trotter_su3", tau, True, "fp64", "su3_constant")
    got = sim.exponentiate(torch.from_numpy(a).cuda()).cpu().numpy()
    assert np.abs(got - orc.exponentiate("one", a, "lie_trotter_su3", tau)).max() < 1e-14 + splitting_tol(0.5, tau)


@pytest.mark.parametrize("tau", [0, 1, 9])
def test_su3_low_tau_factor_structure(ss, tau):
    """Low τ, where the splitting shows: the GPU's factor is the tridiagonalised leapfrog factor of reading R20 and
    U = T^(2^τ) — against the test-side 40-digit construction (W by an mpmath Lanczos process, tests/su3_tridiag_mp.py),
    not against the oracle (a different splitting)."""
    from su3_tridiag_mp import tridiag_factor
    a = W.random_exponent_args_su3(60, 0.5, seed=32)
    sim = ss.Simulator("one", "cf4", "lie_trotter_su3", tau, True, "fp64", "su3_constant")
    got = sim.exponentiate(torch.from_numpy(a).cuda()).cpu().numpy()
    ref = np.array([tridiag_factor(x, tau)[1] for x in a])
    assert np.abs(got - ref).max() < 1e-14


def test_su3_exponentiator_rejects_4_args(ss):
    sim = ss.Simulator("one", "cf4", "lie_trotter_su3", 24, True, "fp64", "constant")
    with pytest.raises(ValueError):
        sim.exponentiate(torch.zeros((3, 4), dtype=torch.float64, device="cuda"))


def test_g1_sweep_parity_small(ss, orc):
    """G1 (su3_drive sweep) at oracle size: 12 strided sweeps × 0.4 ms (K = 400: several scan tiles)."""
    w = W.g1_su3(batch=8192, duration=0.4e-3)
    w = w.with_(sweep=np.ascontiguousarray(w.sweep[::701][:12]), psi0=W.random_states(12, 3, seed=33))
    parity(ss, orc, w)


@pytest.mark.parametrize("frame", [True, False])
def test_su3_constant_parity(ss, orc, frame):
    f = np.array([[2.1e5, -1.3e5, 3.7e5, 0.9e5, -1.7e5, 0.6e5, 1.2e5, -2.2e5],
                  [0.0, 0.0, 2 * np.pi * 7e5, 2 * np.pi * 72, 0.0, 0.0, 0.0, 0.0]])
    w = W.Workload("su3c", "one", "cf4", "lie_trotter_su3", 24, frame, "su3_constant", 0.0, 300e-6, 100e-9, 1e-6,
                   f, W.random_states(2, 3, seed=34))
    parity(ss, orc, w)


def test_su3_expo_on_four_coefficient_field(ss, orc):
    """The su(3) exponentiator on the paper's neural benchmark field (U, V coefficients zero)."""
    w = W.c2_neural(duration=1e-3).with_(expo="lie_trotter_su3", psi0=W.random_states(1, 3, seed=35))
    parity(ss, orc, w)


def test_su3_matches_four_operator_path(ss):
    """On a 4-coefficient field the general exponentiator reduces to the paper's factor: the su(3) and the
    Lie–Trotter kernels agree to rounding on the C2 workload."""
    w = W.c2_neural(duration=2e-3)
    out = []
    for expo in ("lie_trotter", "lie_trotter_su3"):
        sim = ss.Simulator("one", "cf4", expo, 24, True, "fp64", "neural")
        res = sim.evaluate(torch.from_numpy(w.sweep).cuda(), w.t0, w.t1, w.dt_int, w.dt_out,
                           torch.from_numpy(w.psi0).cuda())
        out.append(res.state.cpu().numpy())
    assert np.abs(out[0] - out[1]).max() < 1e-12


def test_su3_drive_resonant_closed_form_gpu(ss):
    """Resonant su3_drive on the GPU against ψ(t) = e^{−iω0 Jz t} e^{−iH' t} ψ0 (closed form; see the oracle pin)."""
    import scipy.linalg as sl
    r2 = 1 / np.sqrt(2)
    JX = r2 * np.array([[0, 1, 0], [1, 0, 1], [0, 1, 0]], complex)
    JY = r2 * np.array([[0, -1j, 0], [1j, 0, -1j], [0, 1j, 0]], complex)
    JZ = np.diag([1.0, 0.0, -1.0]).astype(complex)
    Q = np.diag([1.0, -2.0, 1.0]).astype(complex) / 3
    U1, V1 = JX @ JX - JY @ JY, JX @ JZ + JZ @ JX
    p = W.su3_drive_params(omega_x=2 * np.pi * 3e3, omega_v=2 * np.pi * 1.3e3, omega_u=2 * np.pi * 2e3)
    psi0 = W.random_states(1, 3, seed=36)
    sim = ss.Simulator("one", "cf4", "lie_trotter_su3", 24, True, "fp64", "su3_drive")
    res = sim.evaluate(torch.from_numpy(p[None, :]).cuda(), 0.0, 1e-3, 100e-9, 1e-6, torch.from_numpy(psi0).cuda())
    st = res.state.cpu().numpy()[0]
    w0, wq, Ox, Ov, Ou, _ = p
    Hp = wq * Q + Ox * JX + Ov * V1 + Ou * U1
    ts = np.arange(1001) * 1e-6
    exact = np.array([np.exp(-1j * w0 * np.diag(JZ).real * t) * (sl.expm(-1j * Hp * t) @ psi0[0]) for t in ts])
    assert np.abs(st - exact).max() < 3e-12


@pytest.mark.parametrize("method", ["midpoint", "heun"])
def test_su3_euler_samplers_parity(ss, orc, method):
    w = W.g1_su3(batch=2, duration=0.3e-3).with_(method=method, psi0=W.random_states(2, 3, seed=37))
    parity(ss, orc, w)


def test_su3_fp32_parity(ss, orc):
    w = W.g1_su3(batch=8192, duration=3e-3)
    w = w.with_(sweep=np.ascontiguousarray(w.sweep[::2731][:3]), psi0=W.random_states(3, 3, seed=38))
    parity(ss, orc, w, precision="fp32", tol=TOL32)


@pytest.mark.parametrize("precision,tol", [("fp64", 1e-10), ("fp32", 1e-4)])
def test_su3_user_field_matches_builtin(ss, orc, precision, tol):
    """A user field (NVRTC, 8 coefficients) transcribing su3_drive reproduces the oracle's built-in field, through
    the FP64 kernel and the FP32 float2-lockstep kernel compiled at run time."""
    src = r"""
__device__ void user_field(double t_k, double off, const double* p, double f[8]) {
  const double ph = p[5] * t_k + p[5] * off;     // adequate at t <= 1 ms (reading R8 concerns t ~ 1 s)
  double s, c; sincos(ph, &s, &c);
  double s2, c2; sincos(2.0 * ph, &s2, &c2);
  f[0] = p[2] * c; f[1] = p[2] * s; f[2] = p[0]; f[3] = p[1];
  f[4] = p[4] * c2; f[5] = p[4] * s2; f[6] = p[3] * c; f[7] = p[3] * s;
}"""
    w = W.g1_su3(batch=8192, duration=0.2e-3)
    w = w.with_(sweep=np.ascontiguousarray(w.sweep[::1999][:4]), psi0=W.random_states(4, 3, seed=39))
    sim = ss.Simulator("one", "cf4", "lie_trotter_su3", 24, True, precision, "user", field_source=src, n_params=6)
    res = sim.evaluate(torch.from_numpy(w.sweep).cuda(), w.t0, w.t1, w.dt_int, w.dt_out, torch.from_numpy(w.psi0).cuda())
    st_o, _ = orc.evaluate("one", "cf4", "lie_trotter_su3", 24, True, "su3_drive", sweep=w.sweep, t0=w.t0, t1=w.t1,
                           dt_int=w.dt_int, dt_out=w.dt_out, psi0=w.psi0, want_unitaries=False)
    assert np.abs(res.state.cpu().numpy() - st_o).max() < tol


def test_g1_fullsize_sampled(ss, orc):
    """G1 at full size (8192 sweeps × 10 ms) in the bench's launch configuration; 4 sampled sweeps vs the oracle."""
    w = W.g1_su3()
    sim = ss.Simulator("one", "cf4", "lie_trotter_su3", 24, True, "fp64", "su3_drive")
    res = sim.evaluate(torch.from_numpy(w.sweep).cuda(), w.t0, w.t1, w.dt_int, w.dt_out, torch.from_numpy(w.psi0).cuda(),
                       want_unitaries=False)
    st = res.state
    idx = [0, 2047, 5000, 8191]
    st_o, _ = orc.evaluate("one", "cf4", "lie_trotter_su3", 24, True, "su3_drive", sweep=w.sweep[idx], t0=w.t0,
                           t1=w.t1, dt_int=w.dt_int, dt_out=w.dt_out, psi0=w.psi0[idx], want_unitaries=False)
    assert np.abs(st[idx].cpu().numpy() - st_o).max() < TOL64
    # FP64 chain drift ≲ 2e-16 per interval (measured 1.7e-12 at K = 1e4 for the dense su(3) squarings)
    norms = torch.linalg.vector_norm(st[:, -1], dim=-1)
    assert (norms - 1).abs().max().item() < 1e-15 * w.K
