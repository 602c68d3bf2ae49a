"""Compact SU(2) operators between the interval kernel and the scan: the SU(2)-form paths (spin-half,
analytic spin-one) hand each U_k to the state scan as its SU(2) element (a, b) when U_k is not an output.

* Every scan kernel (cooperative, chain, scan2, scan3) over random SU(2) elements against the oracle's sequential
  long-double chain of the dense matrices — U itself for dim 2, its spin-1 representation D¹(U) (reading R14) for
  dim 3 — element by element, with the fused ⟨J⟩ on some shapes.
* The whole path through ss_evaluate(d_unitaries = NULL) against the oracle, on shapes that route the compact
  operators through each scan kernel, and against the dense path (want_unitaries=True) to rounding.
"""
import numpy as np
import pytest
import torch

import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ss():
    import paper_2204_05586_b200 as ss
    assert torch.cuda.is_available()
    ss.load()
    return ss


def random_su2(B, K, seed):
    """(a, b) of Haar-random SU(2) elements from unit quaternions: [B][K][2] complex128."""
    q = np.random.default_rng(seed).standard_normal((B, K, 4))
    q /= np.linalg.norm(q, axis=-1, keepdims=True)
    return np.stack([q[..., 0] + 1j * q[..., 1], q[..., 2] + 1j * q[..., 3]], -1)


def dense_of(ops, d):
    """The dense operators the compact ones stand for, written from the textbook definitions (not the kernel's):
    U = [[a, b], [−b*, a*]]; for d = 3 the spin-1 representation D¹(U) in the basis m = +1, 0, −1."""
    a, b = ops[..., 0], ops[..., 1]
    if d == 2:
        return np.stack([np.stack([a, b], -1), np.stack([-np.conj(b), np.conj(a)], -1)], -2)
    s2 = np.sqrt(2.0)
    return np.stack([np.stack([a * a, s2 * a * b, b * b], -1),
                     np.stack([-s2 * a * np.conj(b), np.abs(a) ** 2 - np.abs(b) ** 2, s2 * np.conj(a) * b], -1),
                     np.stack([np.conj(b) ** 2, -s2 * np.conj(a) * np.conj(b), np.conj(a) ** 2], -1)], -2)


def test_dense_of_is_a_representation():
    """D¹ as written above is a homomorphism (D¹(xy) = D¹(x)D¹(y)) and unitary — pins the test's own map."""
    x, y = random_su2(1, 50, 1)[0], random_su2(1, 50, 2)[0]
    prod = np.stack([x[:, 0] * y[:, 0] - x[:, 1] * np.conj(y[:, 1]), x[:, 0] * y[:, 1] + x[:, 1] * np.conj(y[:, 0])], -1)
    for d in (2, 3):
        Dx, Dy, Dp = dense_of(x, d), dense_of(y, d), dense_of(prod, d)
        assert np.abs(Dx @ Dy - Dp).max() < 1e-14
        assert np.abs(Dx @ np.conj(np.swapaxes(Dx, -1, -2)) - np.eye(d)).max() < 1e-14


@pytest.mark.parametrize("d", [2, 3])
@pytest.mark.parametrize("B,K,spin", [(1, 1, False), (3, 255, True), (2, 100000, False),   # cooperative scan
                                      (4100, 37, True), (5000, 9, False),                 # per-sweep chain
                                      (520, 20, False), (7, 300000, True),                # scan2 / scan3 (several)
                                      (1, 1300001, False), (1, 8192 * 600, False)])       # scan3 single sweep
def test_scan_su2_vs_sequential_chain(ss, orc, d, B, K, spin):
    if B * K > 4e6 and d == 3:
        K = K // 2 + 1                                   # oracle time: ≤ 2.5e6 long-double 3×3 steps
    ops = random_su2(B, K, seed=B * 7 + K)
    psi0 = W.random_states(B, d, seed=41)
    ref = orc.chain(dense_of(ops, d), psi0)
    st, J = ss.scan_states_su2(torch.from_numpy(ops).cuda(), torch.from_numpy(psi0).cuda(), d, want_spin=spin)
    tol = 1e-12 * max(1.0, np.sqrt(K) / 10)
    assert np.abs(st.cpu().numpy() - ref).max() < tol
    if spin:
        refJ = orc.spin_projection("half" if d == 2 else "one", ref)
        assert np.abs(J.cpu().numpy() - refJ).max() < 2 * tol


def test_scan_su2_spin_only(ss, orc):
    ops = random_su2(3, 5000, seed=5)
    psi0 = W.random_states(3, 3, seed=6)
    ref = orc.spin_projection("one", orc.chain(dense_of(ops, 3), psi0))
    st, J = ss.scan_states_su2(torch.from_numpy(ops).cuda(), torch.from_numpy(psi0).cuda(), 3, want_states=False,
                               want_spin=True)
    assert st is None and np.abs(J.cpu().numpy() - ref).max() < 1e-12


def _run(ss, w, want_unitaries):
    sim = ss.Simulator(w.spin, w.method, w.expo, w.tau, w.frame, "fp64", w.field)
    res = sim.evaluate(torch.from_numpy(w.sweep).cuda(), w.t0, w.t1, w.dt_int, w.dt_out,
                       torch.from_numpy(w.psi0).cuda(), want_unitaries=want_unitaries)
    return res.state.cpu().numpy()


@pytest.mark.parametrize("shape", ["c4_short", "c5_an_short", "half_batch_chain", "half_scan3", "one_an_scan2"])
def test_evaluate_compact_vs_oracle(ss, orc, shape):
    """ss_evaluate without U (compact operators) against the long-double oracle and the dense path."""
    if shape == "c4_short":                 # one sweep, 2e4 intervals: cooperative scan
        w = W.c4_long(duration=0.02)
    elif shape == "c5_an_short":            # analytic spin-one, 3 sweeps × 5000 intervals
        w = W.c5_matrix("analytic", batch=3).with_(t1=0.005)
    elif shape == "half_batch_chain":       # 4100 spin-half sweeps: per-sweep chain kernel
        base = W.c4_long(duration=20e-6, dt_int=10e-9)
        w = base.with_(sweep=np.repeat(base.sweep, 4100, 0) * np.linspace(1.0, 1.02, 4100)[:, None],
                       psi0=W.random_states(4100, 2, seed=44))
    elif shape == "half_scan3":             # one spin-half sweep of 2.5e6 intervals (80 MB compact > L2 bound): scan3
        w = W.c4_long(duration=0.025, dt_int=1e-9, dt_out=10e-9)
    else:                                   # 520 analytic spin-one sweeps × 20 intervals: scan2
        w = W.c5_matrix("analytic", batch=520).with_(t1=20e-6)
    st = _run(ss, w, want_unitaries=False)
    st_dense = _run(ss, w, want_unitaries=True)
    ref = orc.evaluate(w.spin, w.method, w.expo, w.tau, w.frame, w.field, sweep=w.sweep, t0=w.t0, t1=w.t1,
                       dt_int=w.dt_int, dt_out=w.dt_out, psi0=w.psi0)[0]
    assert np.abs(st - ref).max() <= 1e-10, shape
    # two FP64 product orders (different scan kernels / tilings), each drifting ≈ 3e-17 per interval from the exact
    # chain: at most ≈ 6e-17·K apart
    assert np.abs(st - st_dense).max() <= max(1e-12, 6e-17 * w.K), shape


def test_host_api_compact_matches_device(ss):
    """The host-buffer pipeline without U (compact operators in its staging slots) equals the device call to
    rounding (C4 shape: time chunks from a running carry)."""
    w = W.c4_long(duration=0.05)
    sim = ss.Simulator(w.spin, w.method, w.expo, w.tau, w.frame, "fp64", w.field)
    st_d = _run(ss, w, want_unitaries=False)
    for chunks in (0, 1, 6):
        st_h, U_h = sim.evaluate_host(w.sweep, w.t0, w.t1, w.dt_int, w.dt_out, w.psi0, want_unitaries=False,
                                      n_chunks=chunks)
        assert U_h is None and np.abs(st_h - st_d).max() <= 1e-12


@pytest.mark.parametrize("path", ["coop", "scan2", "scan3", "twopass", "chain"])
@pytest.mark.parametrize("d,compact", [(2, True), (3, True), (2, False), (3, False)])
def test_every_scan_path_forced(ss, orc, monkeypatch, path, d, compact):
    """SPINSIM_SCAN_PATH forces each scan kernel (the heuristic picks one per shape): every kernel, for both operator
    formats and both state dimensions, on one shape with ragged tiles and several sweeps, with the fused ⟨J⟩."""
    B, K = 3, 9000 + 37
    psi0 = W.random_states(B, d, seed=51)
    if compact:
        ops = random_su2(B, K, seed=52)
        dense = dense_of(ops, d)
    else:
        dense = dense_of(random_su2(B, K, seed=52), d) * np.exp(1j * np.random.default_rng(53).uniform(
            0, 2 * np.pi, (B, K, 1, d)))                   # unitary, not in the image of D¹
    ref = orc.chain(dense, psi0)
    refJ = orc.spin_projection("half" if d == 2 else "one", ref)
    monkeypatch.setenv("SPINSIM_SCAN_PATH", path)
    pg = torch.from_numpy(psi0).cuda()
    if compact:
        st, J = ss.scan_states_su2(torch.from_numpy(ops).cuda(), pg, d, want_spin=True)
    else:
        st, J = ss.scan_states_spin(torch.from_numpy(dense).cuda(), pg, want_states=True)
    assert np.abs(st.cpu().numpy() - ref).max() < 1e-12
    assert np.abs(J.cpu().numpy() - refJ).max() < 2e-12


@pytest.mark.parametrize("d", [2, 3])
@pytest.mark.parametrize("B,K,forced", [(3, 9000 + 36, True),         # runs of 4 (K = 4·2259)
                                        (2, 8192 + 64, True),         # runs of 32, several warps per sweep
                                        (3, 800_000, False)])         # 77 MB of operators: the heuristic's choice
def test_two_pass_compact_scan(ss, orc, monkeypatch, d, B, K, forced):
    """The standalone two-pass scan of compact operators (run products, coarse scan, run chain) against the oracle's
    sequential chain, with the fused ⟨J⟩; forced, or chosen by the heuristic for a problem beyond the L2 bound."""
    if forced:
        monkeypatch.setenv("SPINSIM_SCAN_PATH", "twopass")
    else:
        monkeypatch.delenv("SPINSIM_SCAN_PATH", raising=False)
    ops = random_su2(B, K, seed=61 + K)
    psi0 = W.random_states(B, d, seed=62)
    ref = orc.chain(dense_of(ops, d), psi0)
    refJ = orc.spin_projection("half" if d == 2 else "one", ref)
    n0 = ss.kernel_launches()
    st, J = ss.scan_states_su2(torch.from_numpy(ops).cuda(), torch.from_numpy(psi0).cuda(), d, want_spin=True)
    assert ss.kernel_launches() - n0 >= 3                   # run products, coarse scan, run chain
    tol = 1e-12 * max(1.0, np.sqrt(K) / 10)
    assert np.abs(st.cpu().numpy() - ref).max() < tol
    assert np.abs(J.cpu().numpy() - refJ).max() < 2 * tol
