"""GPU parity of the advisory Magnus-convergence diagnostic (ss_magnus_bound) against the
long-double oracle: per sweep, the largest Gauss–Legendre estimate of ∫‖H‖₂ over a fine step in the integration
frame, for both spins, all field families, frame on and off."""
import numpy as np
import pytest
import torch

import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ss():
    import paper_2204_05586_b200 as ss
    ss.load()
    return ss


CASES = {
    "c1": lambda: W.c1_rabi("rabi_circular").with_(t1=50e-6),
    "c1_lin_off": lambda: W.c1_rabi("rabi_linear").with_(t1=50e-6, frame=False),
    "c2": lambda: W.c2_neural(duration=0.3e-3),
    "c3": lambda: W.c3_batched(batch=5, duration=0.1e-3).with_(sweep=W.c3_sweep_params()[::1700][:5]),
    "g1": lambda: W.g1_su3(batch=3, duration=0.1e-3),
    "su3c_off": lambda: W.Workload("su3c", "one", "cf4", "lie_trotter_su3", 24, False, "su3_constant", 0.0, 20e-6,
                                   100e-9, 1e-6, np.array([[2.1e5, -1.3e5, 3.7e5, 0.9e5, -1.7e5, 0.6e5, 1.2e5, -2.2e5]]),
                                   W.basis_state(3)),
    "half_const": lambda: W.Workload("hc", "half", "cf4", "analytic", 24, False, "constant", 0.0, 4e-6, 2e-7, 4e-7,
                                     np.array([[4 * np.pi * 1e6, 0.0, 0.0, 0.0]]), W.basis_state(2)),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_magnus_bound_parity(ss, orc, name):
    w = CASES[name]()
    sim = ss.Simulator(w.spin, w.method, w.expo, w.tau, w.frame, "fp64", w.field)
    got = sim.magnus_bound(torch.from_numpy(np.ascontiguousarray(w.sweep)).cuda(), w.t0, w.t1, w.dt_int,
                           w.dt_out).cpu().numpy()
    ref = orc.magnus_bound(w.spin, w.frame, w.field, sweep=w.sweep, t0=w.t0, t1=w.t1, dt_int=w.dt_int,
                           dt_out=w.dt_out)
    assert np.all(np.abs(got - ref) <= 1e-11 * ref + 1e-300), (got, ref)


def test_magnus_threshold_example(ss):
    """‖H‖₂ = 2π·1e6 rad/s at δt = 100 ns gives 0.628 < ξ, at 200 ns 1.257 > ξ."""
    from paper_2204_05586_b200._lib import SS_MAGNUS_XI
    sim = ss.Simulator("half", "cf4", "analytic", 24, False, "fp64", "constant")
    sweep = torch.tensor([[4 * np.pi * 1e6, 0.0, 0.0, 0.0]], dtype=torch.float64, device="cuda")
    a = sim.magnus_bound(sweep, 0.0, 4e-6, 1e-7, 4e-7).item()
    b = sim.magnus_bound(sweep, 0.0, 4e-6, 2e-7, 4e-7).item()
    assert a == pytest.approx(0.2 * np.pi, rel=1e-14) and a < SS_MAGNUS_XI
    assert b == pytest.approx(0.4 * np.pi, rel=1e-14) and b > SS_MAGNUS_XI


def test_magnus_bound_user_field(ss, orc):
    """The diagnostic through a run-time compiled (NVRTC) user field equals the built-in field's (same Eq.
    neural_pulse transcription) and the oracle's."""
    src = r"""
__device__ void user_field(double t_k, double off, const double* p, double f[4]) {
  const double t = t_k + off;
  f[0] = 2.0 * p[2] * cos(p[1] * t);
  const double x = p[4] * ((t_k - p[5]) + off);
  f[2] = p[0] + p[3] * ((x >= 0.0 && x <= 6.283185307179586) ? sin(x) : 0.0);
  f[3] = p[6];
}"""
    w = W.c2_neural(duration=0.2e-3).with_(sweep=W.neural_params(t_p=0.05e-3)[None, :])
    sim_u = ss.Simulator("one", "cf4", "lie_trotter", 24, True, "fp64", "user", field_source=src, n_params=7)
    sim_b = ss.Simulator("one", "cf4", "lie_trotter", 24, True, "fp64", "neural")
    sw = torch.from_numpy(w.sweep).cuda()
    mu = sim_u.magnus_bound(sw, w.t0, w.t1, w.dt_int, w.dt_out).item()
    mb = sim_b.magnus_bound(sw, w.t0, w.t1, w.dt_int, w.dt_out).item()
    ref = orc.magnus_bound("one", True, "neural", sweep=w.sweep, t0=w.t0, t1=w.t1, dt_int=w.dt_int, dt_out=w.dt_out)[0]
    assert mu == pytest.approx(ref, rel=1e-9) and mb == pytest.approx(ref, rel=1e-11)
