"""User-defined field functions compiled at run time (the paper's user field functions
P:643-650): parity with the oracle's built-in field of the same formula, exactness where CF4 is exact, error paths."""
import numpy as np
import pytest
import torch

import workloads as W

pytestmark = pytest.mark.gpu

NEURAL_SRC = r"""
__device__ void user_field(double t_k, double off, const double* p, double f[4]) {
  // Eq. neural_pulse (P:681) with p = [w_bias, w_rf, Omega, Omega_p, w_sig, t_p, w_q]
  const double t = t_k + off;
  f[0] = 2.0 * p[2] * cos(p[1] * t);
  const double x = p[4] * ((t_k - p[5]) + off);
  f[2] = p[0] + ((x >= 0.0 && x <= 6.283185307179586) ? p[3] * sin(x) : 0.0);
  f[3] = p[6];
}
"""

CHIRP_SRC = r"""
__device__ void user_field(double t_k, double off, const double* p, double f[4]) {
  f[2] = p[0] + p[1] * (t_k + off);        // linear chirp of the bias: w_z(t) = w0 + beta t
}
"""


@pytest.fixture(scope="module")
def ss():
    import paper_2204_05586_b200 as ss
    ss.load()
    return ss


@pytest.mark.parametrize("spin", ["half", "one"])
def test_user_field_matches_builtin_formula(ss, orc, spin):
    w = W.c2_neural(duration=2e-3).with_(spin=spin, expo="analytic" if spin == "half" else "lie_trotter",
                                         sweep=W.neural_params(t_p=0.5e-3, omega_q=0.0 if spin == "half" else W.OMEGA_Q)[None, :],
                                         psi0=W.random_states(1, 2 if spin == "half" else 3, seed=40))
    sim = ss.Simulator(w.spin, w.method, w.expo, w.tau, w.frame, "fp64", "user", field_source=NEURAL_SRC, n_params=7)
    res = sim.evaluate(torch.from_numpy(w.sweep).cuda(), w.t0, w.t1, w.dt_int, w.dt_out, torch.from_numpy(w.psi0).cuda())
    st_o, U_o = orc.evaluate(w.spin, w.method, w.expo, w.tau, w.frame, "neural", sweep=w.sweep, t0=w.t0, t1=w.t1,
                             dt_int=w.dt_int, dt_out=w.dt_out, psi0=w.psi0)
    assert np.abs(res.time_evolution.cpu().numpy() - U_o).max() <= 1e-10
    assert np.abs(res.state.cpu().numpy() - st_o).max() <= 1e-10


@pytest.mark.parametrize("method", ["cf4", "midpoint"])
def test_user_chirp_exact(ss, method):
    """Commuting linear ω_z(t): CF4's Gauss points (and the midpoint rule) integrate it exactly, so
    U_k = exp(−i Jz ∫ω_z) = diag(e^{∓iΘ/2}), Θ = ω0 Δt + β (t_{k+1}² − t_k²)/2, frame off."""
    w0, beta = 2 * np.pi * 1e5, 2 * np.pi * 3e7
    sim = ss.Simulator("half", method, "analytic", 24, False, "fp64", "user", field_source=CHIRP_SRC, n_params=2)
    sweep = torch.tensor([[w0, beta]], dtype=torch.float64).cuda()
    psi0 = torch.tensor([[1, 0]], dtype=torch.complex128).cuda()
    res = sim.evaluate(sweep, 0.0, 50e-6, 250e-9, 1e-6, psi0)
    U = res.time_evolution[0].cpu().numpy()
    k = np.arange(50)
    t0, t1 = k * 1e-6, (k + 1) * 1e-6
    theta = w0 * 1e-6 + beta * (t1 ** 2 - t0 ** 2) / 2
    assert np.abs(U[:, 0, 0] - np.exp(-0.5j * theta)).max() < 1e-13
    assert np.abs(U[:, 1, 1] - np.exp(0.5j * theta)).max() < 1e-13
    assert np.abs(U[:, 0, 1]).max() == 0.0


def test_user_field_errors(ss):
    with pytest.raises(ss.SpinsimError, match="compilation failed"):
        ss.Simulator("half", field="user", field_source="__device__ void user_field( {", n_params=1)
    with pytest.raises(ss.SpinsimError):
        ss.Simulator("one", "cf4", "analytic", field="user", field_source=CHIRP_SRC, n_params=2)
