"""Full-size verification runs (part of the default -m gpu suite): the complete BASELINE workloads on the GPU
against the complete long-double oracle run on every host core (≈ 1–2 min of CPU in total on a 16-core host).

C4 is where FP64 drift matters (1e9 fine steps, SURVEY [V16]): every one of its 1e6 + 1 states is compared.
"""
import time

import numpy as np
import pytest
import torch

import workloads as W

pytestmark = pytest.mark.gpu


def _run(w):
    import paper_2204_05586_b200 as ss
    sim = ss.Simulator(w.spin, w.method, w.expo, w.tau, w.frame, "fp64", w.field)
    res = sim.evaluate(torch.from_numpy(w.sweep).cuda(), w.t0, w.t1, w.dt_int, w.dt_out,
                       torch.from_numpy(w.psi0).cuda(), want_unitaries=False)
    torch.cuda.synchronize()
    return res.state.cpu().numpy()


def test_c4_every_state_vs_full_oracle(orc):
    """C4 complete: 1 s at δt = 1 ns (1e9 fine steps), every one of the 1e6 + 1 states vs the long-double oracle."""
    w = W.c4_long()
    st_g = _run(w)
    t = time.perf_counter()
    st_o, _ = orc.evaluate(w.spin, w.method, w.expo, w.tau, w.frame, w.field, sweep=w.sweep, t0=w.t0, t1=w.t1,
                           dt_int=w.dt_int, dt_out=w.dt_out, psi0=w.psi0, want_unitaries=False)
    err = np.abs(st_g - st_o).max(axis=(0, 2))
    print(f"\nC4 full: oracle {time.perf_counter() - t:.0f} s; max |dpsi| over all {st_g.shape[1]} states = "
          f"{err.max():.3e} (at t = {err.argmax() * w.dt_out:.4f} s); at t = 0.1/0.5/1 s: "
          f"{err[100000]:.2e} / {err[500000]:.2e} / {err[-1]:.2e}; norm drift {abs(np.linalg.norm(st_g[0, -1]) - 1):.2e}")
    assert err.max() <= 1e-10


def test_c3_sampled_sweeps_every_state(orc):
    """C3 complete GPU run; 32 sweeps (strided over the 8192) compared state by state with the oracle."""
    w = W.c3_batched()
    st_g = _run(w)
    idx = np.linspace(0, w.batch - 1, 32).astype(int)
    st_o, _ = orc.evaluate(w.spin, w.method, w.expo, w.tau, w.frame, w.field, sweep=w.sweep[idx], t0=w.t0, t1=w.t1,
                           dt_int=w.dt_int, dt_out=w.dt_out, psi0=w.psi0[idx], want_unitaries=False)
    err = np.abs(st_g[idx] - st_o).max()
    print(f"\nC3: 32 sweeps x 10001 states: max |dpsi| = {err:.3e}")
    assert err <= 1e-10


def test_g1_sampled_sweeps_every_state(orc):
    """G1 (general spin-one, su(3) Lie–Trotter) complete GPU run; 32 sweeps compared state by state with the oracle."""
    w = W.g1_su3()
    st_g = _run(w)
    idx = np.linspace(0, w.batch - 1, 32).astype(int)
    st_o, _ = orc.evaluate(w.spin, w.method, w.expo, w.tau, w.frame, w.field, sweep=w.sweep[idx], t0=w.t0, t1=w.t1,
                           dt_int=w.dt_int, dt_out=w.dt_out, psi0=w.psi0[idx], want_unitaries=False)
    err = np.abs(st_g[idx] - st_o).max()
    print(f"\nG1: 32 sweeps x {st_g.shape[1]} states: max |dpsi| = {err:.3e}")
    assert err <= 1e-10
