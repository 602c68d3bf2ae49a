"""GPU parity: the CUDA path (through the C ABI) against the long-double oracle on the same seeded inputs.

Bar (BASELINE.json north_star): max |ψ_gpu − ψ_oracle| ≤ 1e-10 in FP64, ≤ 1e-4 in FP32 mode, element by element over
every (sweep, k, component) — and the same for the interval unitaries U_k.  Full BASELINE sizes are covered in
test_gpu_fullsize.py on sampled outputs.
"""
import numpy as np
import pytest
import torch

import workloads as W

pytestmark = pytest.mark.gpu

TOL64 = 1e-10
TOL32 = 1e-4


@pytest.fixture(scope="module")
def ss():
    import paper_2204_05586_b200 as ss
    assert torch.cuda.is_available()
    ss.load()
    return ss


def gpu_run(ss, w: W.Workload, precision="fp64", want_unitaries=True):
    sim = ss.Simulator(w.spin, w.method, w.expo, w.tau, w.frame, precision, w.field)
    sweep = torch.from_numpy(np.ascontiguousarray(w.sweep)).cuda()
    psi0 = torch.from_numpy(np.ascontiguousarray(w.psi0)).cuda()
    res = sim.evaluate(sweep, w.t0, w.t1, w.dt_int, w.dt_out, psi0, want_unitaries=want_unitaries)
    torch.cuda.synchronize()
    U = res.time_evolution.cpu().numpy() if want_unitaries else None
    return res.state.cpu().numpy(), U


def oracle_run(orc, w: W.Workload, **kw):
    return orc.evaluate(w.spin, w.method, w.expo, w.tau, w.frame, w.field, sweep=w.sweep, t0=w.t0, t1=w.t1,
                        dt_int=w.dt_int, dt_out=w.dt_out, psi0=w.psi0, **kw)


def assert_parity(ss, orc, w, tol=TOL64, precision="fp64"):
    st_g, U_g = gpu_run(ss, w, precision)
    st_o, U_o = oracle_run(orc, w)
    eU = np.abs(U_g - U_o).max()
    eS = np.abs(st_g - st_o).max()
    assert eU <= tol and eS <= tol, (w.name, precision, eU, eS)
    return eU, eS


# ---- building blocks -------------------------------------------------------------------------------------------
@pytest.mark.parametrize("spin,expo,scale", [("half", "analytic", 1.0), ("half", "analytic", 1e-6),
                                             ("one", "lie_trotter", 1.0), ("one", "lie_trotter", 1e-6),
                                             # around the second-order Taylor bound of the factor (2^-27, §5 item 9)
                                             ("one", "lie_trotter", 0.03), ("one", "lie_trotter", 0.02),
                                             ("one", "analytic", 1.0)])
def test_exponentiator_parity(ss, orc, spin, expo, scale):
    a = W.random_exponent_args(5000, scale, seed=21, quad=(expo != "analytic" or spin == "half"))
    if spin == "half" or expo == "analytic":
        a[:, 3] = 0.0
    a[:3] = 0.0                                       # exact zero args (reading R3/R4)
    a[3, :2] = 0.0                                    # Φ = 0 with z, q ≠ 0
    sim = ss.Simulator(spin, "cf4", expo, 24, True, "fp64", "constant")
    got = sim.exponentiate(torch.from_numpy(a).cuda()).cpu().numpy()
    ref = orc.exponentiate(spin, a, expo, 24)
    assert np.abs(got - ref).max() <= 4e-16 * max(1.0, scale) * 8
    sim32 = ss.Simulator(spin, "cf4", expo, 24, True, "fp32", "constant")
    got32 = sim32.exponentiate(torch.from_numpy(a).cuda()).cpu().numpy()
    assert np.abs(got32 - ref).max() <= 2e-6


@pytest.mark.parametrize("tau", [0, 1, 7, 24, 40])
def test_lie_trotter_tau_parity(ss, orc, tau):
    a = W.random_exponent_args(500, 0.5, seed=22)
    sim = ss.Simulator("one", "cf4", "lie_trotter", tau, True, "fp64", "constant")
    got = sim.exponentiate(torch.from_numpy(a).cuda()).cpu().numpy()
    assert np.abs(got - orc.exponentiate("one", a, "lie_trotter", tau)).max() < 1e-14


# ---- configs at oracle-friendly sizes (several scan tiles + ragged tails) ---------------------------------------
@pytest.mark.parametrize("field", ["rabi_circular", "rabi_linear"])
def test_c1_rabi_parity(ss, orc, field):
    assert_parity(ss, orc, W.c1_rabi(field))


def test_c2_neural_parity_short(ss, orc):
    assert_parity(ss, orc, W.c2_neural(duration=3.3e-3))            # K = 3300: 13 tiles of 256, ragged tail


@pytest.mark.parametrize("dt_int", [1e-6, 250e-9, 10e-9])
def test_c2_dt_sweep_parity(ss, orc, dt_int):
    assert_parity(ss, orc, W.c2_neural(dt_int=dt_int, duration=0.2e-3 if dt_int < 1e-7 else 1e-3))


def test_c3_batched_parity_small(ss, orc):
    w = W.c3_batched(batch=24, duration=0.5e-3)
    w = w.with_(sweep=W.c3_sweep_params()[::341][:24], psi0=W.random_states(24, 3, seed=23))
    assert_parity(ss, orc, w)


def test_c4_spin_half_parity_short(ss, orc):
    assert_parity(ss, orc, W.c4_long(duration=2e-3).with_(sweep=W.neural_params(t_p=1e-3, omega_q=0.0)[None, :]))


@pytest.mark.parametrize("spin,method", [("half", "midpoint"), ("one", "cf4"), ("one", "heun")])
def test_short_su2_series_parity(ss, orc, spin, method):
    """1 ns steps put every SU(2) exponential below the per-interval bound r ≤ 2^-13 (two-term series, DESIGN.md §5
    item 15) — spin-half with a midpoint sampler and the analytic spin-one path (ω_q = 0)."""
    w = W.c4_long(duration=0.4e-3).with_(spin=spin, method=method, expo="analytic",
                                         sweep=W.neural_params(t_p=0.2e-3, omega_q=0.0)[None, :],
                                         psi0=W.random_states(1, 2 if spin == "half" else 3, seed=27))
    assert_parity(ss, orc, w)


@pytest.mark.parametrize("expo", ["lie_trotter", "analytic"])
def test_c5_parity_short(ss, orc, expo):
    w = W.c5_matrix(expo, batch=3)
    assert_parity(ss, orc, w.with_(t1=2e-3))


@pytest.mark.parametrize("spin,expo", [("one", "lie_trotter"), ("one", "analytic"), ("half", "analytic")])
def test_fp32_mode_parity(ss, orc, spin, expo):
    w = W.c5_matrix(expo, batch=2).with_(t1=5e-3)
    if spin == "half":
        w = w.with_(spin="half", psi0=W.basis_state(2, 2))
    assert_parity(ss, orc, w, tol=TOL32, precision="fp32")


@pytest.mark.parametrize("method", ["midpoint", "heun"])
@pytest.mark.parametrize("spin", ["half", "one"])
def test_euler_samplers_parity(ss, orc, method, spin):
    w = W.c2_neural(duration=0.5e-3).with_(method=method, spin=spin, expo="analytic" if spin == "half" else "lie_trotter",
                                           psi0=W.random_states(1, 2 if spin == "half" else 3, seed=24))
    assert_parity(ss, orc, w)


@pytest.mark.parametrize("frame", [True, False])
@pytest.mark.parametrize("field,params", [
    ("constant", [2.1e5, -1.3e5, 3.7e5, 0.9e5]),
    ("gradient", [3.0e5, 0.4e5]),
    ("rabi_circular", [2 * np.pi * 700e3, 2 * np.pi * 1e3]),
])
def test_fields_and_frame_parity(ss, orc, field, params, frame):
    w = W.Workload("f", "one", "cf4", "lie_trotter", 24, frame, field, 0.0, 0.3e-3, 100e-9, 1e-6,
                   np.array([params], float), W.random_states(1, 3, seed=25))
    assert_parity(ss, orc, w)


# ---- edge cases ------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("K,L", [(1, 1), (1, 7), (2, 1), (255, 2), (256, 1), (257, 1), (513, 1), (1000, 3)])
def test_grid_edge_cases(ss, orc, K, L):
    for spin in ("half", "one"):
        w = W.c2_neural(dt_int=1e-6 / L).with_(t1=K * 1e-6, spin=spin,
                                               expo="analytic" if spin == "half" else "lie_trotter",
                                               psi0=W.random_states(2, 2 if spin == "half" else 3, seed=26),
                                               sweep=np.stack([W.neural_params(t_p=0.1e-3)] * 2))
        assert_parity(ss, orc, w)


def test_time_start_nonzero_and_large(ss, orc):
    """Large t (RF phase ≈ 4.4e6 rad): the per-interval double-double phase reduction (reading R8)."""
    w = W.c4_long(duration=0.1).with_(t0=0.9, t1=0.9 + 0.2e-3, dt_int=10e-9,
                                      sweep=W.neural_params(t_p=0.90005, omega_q=0.0)[None, :])
    assert_parity(ss, orc, w)


def test_validation_errors(ss):
    from paper_2204_05586_b200._lib import SS_ERR_INVALID, SS_ERR_NONFINITE
    sim = ss.Simulator("one", "cf4", "analytic", 24, True, "fp64", "neural")
    sweep = torch.from_numpy(W.neural_params()[None, :]).cuda()          # ω_q ≠ 0
    psi0 = torch.from_numpy(W.basis_state(3)).cuda()
    with pytest.raises(ss.SpinsimError) as e:
        sim.evaluate(sweep, 0.0, 1e-5, 1e-7, 1e-6, psi0)
    assert e.value.code == SS_ERR_INVALID
    sim2 = ss.Simulator("one")
    bad = sweep.clone()
    bad[0, 2] = float("nan")
    with pytest.raises(ss.SpinsimError) as e:
        sim2.evaluate(bad, 0.0, 1e-5, 1e-7, 1e-6, psi0)
    assert e.value.code == SS_ERR_NONFINITE


# ---- scan, aggregate, carry, projection against the oracle's sequential chain ----------------------------------
def _random_unitaries(B, K, d, seed):
    rng = np.random.default_rng(seed)
    z = rng.standard_normal((B, K, d, d)) + 1j * rng.standard_normal((B, K, d, d))
    q, r = np.linalg.qr(z)
    return q * (np.diagonal(r, axis1=-2, axis2=-1) / np.abs(np.diagonal(r, axis1=-2, axis2=-1)))[..., None, :]


@pytest.mark.parametrize("d", [2, 3])
@pytest.mark.parametrize("B,K", [(1, 1), (3, 255), (2, 256), (5, 1031), (1, 20000), (300, 7),
                                 (4096, 1), (4100, 37), (4097, 8), (5000, 9),    # B >= 4096: per-sweep chain kernel
                                 (2304, 269), (2400, 37), (2303, 40)])   # dense spin-one: chain from 2304 sweeps,
                                                                         # rings of 7–8 stages wrapped ≥ 2× at K = 269
def test_scan_vs_sequential_chain(ss, orc, d, B, K):
    U = _random_unitaries(B, K, d, seed=B * 1000 + K)
    psi0 = W.random_states(B, d, seed=27)
    ref, agg = orc.chain(U, psi0, want_aggregate=True)
    Ug = torch.from_numpy(U).cuda()
    got = ss.scan_states(Ug, torch.from_numpy(psi0).cuda()).cpu().numpy()
    assert np.abs(got - ref).max() < 1e-12 * max(1.0, np.sqrt(K) / 10)
    A = ss.chain_aggregate(Ug).cpu().numpy()
    assert np.abs(A - agg).max() < 1e-12 * max(1.0, np.sqrt(K) / 10)


def _fast_unitaries(B, K, d, seed):
    """Random unitaries without a batched QR (large K): SU(2) from a unit quaternion; for d = 3 the spin-1
    representation of it times random diagonal phases (still unitary, entries all non-trivial)."""
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((B, K, 4))
    q /= np.linalg.norm(q, axis=-1, keepdims=True)
    a, b = q[..., 0] + 1j * q[..., 1], q[..., 2] + 1j * q[..., 3]
    if d == 2:
        return np.stack([np.stack([a, -np.conj(b)], -1), np.stack([b, np.conj(a)], -1)], -2)
    s2 = np.sqrt(2.0)
    u = np.stack([np.stack([a * a, -s2 * a * np.conj(b), np.conj(b) ** 2], -1),
                  np.stack([s2 * a * b, np.abs(a) ** 2 - np.abs(b) ** 2, -s2 * np.conj(a) * np.conj(b)], -1),
                  np.stack([b * b, s2 * np.conj(a) * b, np.conj(a) ** 2], -1)], -2)
    return u * np.exp(1j * rng.uniform(0, 2 * np.pi, (B, K, 1, 3)))


@pytest.mark.parametrize("d,B,K", [(3, 1, 1422 * 128), (3, 1, 1422 * 128 + 1),   # 204 768 B per CTA: staged / not
                                   (2, 1, 3200 * 128), (2, 1, 3200 * 128 + 1),   # 204 800 B per CTA: staged / not
                                   (3, 1, 100000), (3, 2, 100000), (2, 1, 777)])  # C2 shape; 256 CTAs: L2 path
def test_scan_coop_staging_boundary(ss, orc, d, B, K):
    """The cooperative scan stages each CTA's run of operators in shared memory (one bulk copy) when every CTA has an
    SM of its own and the run fits 200 KB, else it reads them through L2: both sides of each bound against the
    oracle's sequential long-double chain."""
    U = _fast_unitaries(B, K, d, seed=K + 7 * B)
    psi0 = W.random_states(B, d, seed=35)
    ref = orc.chain(U, psi0)
    got = ss.scan_states(torch.from_numpy(U).cuda(), torch.from_numpy(psi0).cuda()).cpu().numpy()
    assert np.abs(got - ref).max() < 1e-12 * max(1.0, np.sqrt(K) / 10)


@pytest.mark.parametrize("d,B,K,spin", [(2, 1, 8192 * 600, False),      # tiles of 8192, all full (tensor TMA only)
                                        (2, 1, 1300001, True),          # nst = 4, ragged last tile
                                        (2, 7, 300000, False),          # several sweeps, j-major look-back
                                        (3, 1, 4096 * 592, True),       # tiles of 4096, all full
                                        (3, 3, 700001, False),          # nst = 8, ragged, several sweeps
                                        (3, 1, 600001, True)])          # > 64 MB, < 4 stages per tile: scan2
def test_scan_large_single_sweep_path(ss, orc, d, B, K, spin):
    """Sizes that select the super-tile scan (scan3: tensor-TMA stage boxes, one look-back per tile) — and, last, the
    round-1 tile scan (scan2), which the cooperative scan left to single sweeps past the L2-sized bound — against the
    oracle's sequential long-double chain, element by element; with the fused ⟨J⟩ where `spin`."""
    U = _fast_unitaries(B, K, d, seed=K + B)
    psi0 = W.random_states(B, d, seed=33)
    ref = orc.chain(U, psi0)
    tol = 1e-12 * np.sqrt(K) / 10
    Ug, pg = torch.from_numpy(U).cuda(), torch.from_numpy(psi0).cuda()
    if spin:
        st, J = ss.scan_states_spin(Ug, pg, want_states=True)
        refJ = orc.spin_projection("half" if d == 2 else "one", ref)
        assert np.abs(J.cpu().numpy() - refJ).max() < 2 * tol
    else:
        st = ss.scan_states(Ug, pg)
    assert np.abs(st.cpu().numpy() - ref).max() < tol


def test_compose_carry(ss, orc):
    d, B, G = 3, 4, 5
    A = _random_unitaries(G, B, d, seed=28)           # [G][B][d][d]
    psi0 = W.random_states(B, d, seed=29)
    Ag = torch.from_numpy(A).cuda()
    for part in range(G):
        got = ss.compose_carry(Ag, torch.from_numpy(psi0).cuda(), part).cpu().numpy()
        ref = orc.chain(np.transpose(A[:part], (1, 0, 2, 3)), psi0)[:, -1] if part else psi0
        assert np.abs(got - ref).max() < 1e-14


@pytest.mark.parametrize("spin", ["half", "one"])
def test_spin_projection_parity(ss, orc, spin):
    d = 2 if spin == "half" else 3
    psi = W.random_states(1000, d, seed=30)
    got = ss.spin_projection(spin, torch.from_numpy(psi).cuda()).cpu().numpy()
    assert np.abs(got - orc.spin_projection(spin, psi)).max() < 1e-15


# ---- properties ------------------------------------------------------------------------------------------------
def test_determinism_bitwise(ss):
    w = W.c3_batched(batch=64, duration=0.3e-3)
    a, Ua = gpu_run(ss, w)
    b, Ub = gpu_run(ss, w)
    assert np.array_equal(a, b) and np.array_equal(Ua, Ub)


def test_host_api_matches_device_api(ss):
    w = W.c3_batched(batch=5, duration=0.2e-3)
    st_d, U_d = gpu_run(ss, w)
    sim = ss.Simulator(w.spin, w.method, w.expo, w.tau, w.frame, "fp64", w.field)
    for chunks in (1, 3, 7, 10):                      # geometric chunking incl. more chunks than halvings
        st_h, U_h = sim.evaluate_host(w.sweep, w.t0, w.t1, w.dt_int, w.dt_out, w.psi0, want_unitaries=True,
                                      n_chunks=chunks)
        assert np.array_equal(st_h, st_d) and np.array_equal(U_h, U_d)


def test_host_api_time_chunks_match_device_api(ss):
    """Large batches (≥ 4096 sweeps) pipeline the host-buffer call over time chunks started from a running carry:
    the per-sweep chain scan is sequential, so states and operators equal one device evaluate() bit for bit."""
    w = W.c3_batched(batch=4096, duration=0.2e-3)
    st_d, U_d = gpu_run(ss, w)
    sim = ss.Simulator(w.spin, w.method, w.expo, w.tau, w.frame, "fp64", w.field)
    for chunks in (6, 10, 50):                      # 50: K = 200 = 4·50, chunks of 1–5 intervals
        st_h, U_h = sim.evaluate_host(w.sweep, w.t0, w.t1, w.dt_int, w.dt_out, w.psi0, want_unitaries=True,
                                      n_chunks=chunks)
        assert np.array_equal(st_h, st_d) and np.array_equal(U_h, U_d)


def test_host_api_time_chunks_long_sweep(ss):
    """A single long sweep (C4: 1e6 intervals, ≥ 6 waves of interval work per chunk) also takes the time-chunked host
    pipeline: the operators are bit-identical to the device call, the states equal to rounding (the scan restarts
    from the carry)."""
    w = W.c4_long()
    st_d, U_d = gpu_run(ss, w)
    sim = ss.Simulator(w.spin, w.method, w.expo, w.tau, w.frame, "fp64", w.field)
    for chunks in (6, 8):
        st_h, U_h = sim.evaluate_host(w.sweep, w.t0, w.t1, w.dt_int, w.dt_out, w.psi0, want_unitaries=True,
                                      n_chunks=chunks)
        assert np.array_equal(U_h, U_d)
        # two FP64 product orders over 1e6 intervals: each drifts ≈ 3e-11 from the exact chain (SURVEY §0.7,
        # profiles/r01/long_verification*.txt); measured difference 5.5e-13
        assert np.abs(st_h - st_d).max() <= 1e-11


@pytest.mark.parametrize("batch", [1, 3])
def test_host_api_wave_pair_c2(ss, batch):
    """The paper's benchmark shape (C2: 1e5 intervals per sweep, 2.6 waves of interval work for one sweep) takes the
    wave-aligned two-chunk host pipeline: operators bit-identical to the device call, states equal to rounding (the
    scan restarts from the carry at the chunk boundary)."""
    w = W.c2_neural()
    if batch > 1:
        w = w.with_(sweep=np.repeat(w.sweep, batch, axis=0) * np.linspace(1.0, 1.01, batch)[:, None],
                    psi0=W.random_states(batch, 3, seed=33))
    n0 = ss.kernel_launches()
    st_d, U_d = gpu_run(ss, w)
    n_dev = ss.kernel_launches() - n0
    sim = ss.Simulator(w.spin, w.method, w.expo, w.tau, w.frame, "fp64", w.field)
    for chunks in (0, 40):
        n0 = ss.kernel_launches()
        st_h, U_h = sim.evaluate_host(w.sweep, w.t0, w.t1, w.dt_int, w.dt_out, w.psi0, want_unitaries=True,
                                      n_chunks=chunks)
        assert ss.kernel_launches() - n0 > n_dev        # two chunks: interval + scan launches for each
        assert np.array_equal(U_h, U_d)
        # two FP64 product orders over 1e5 spin-one intervals (each ≈ 5e-12 from the exact chain, §9.0c)
        assert np.abs(st_h - st_d).max() <= 1e-11


@pytest.mark.parametrize("which", ["C4", "C2", "G1"])
def test_partition_reproduces_unitaries_bitwise(ss, which):
    """The time grid uses the global k (and the sub-interval split is chosen from the whole problem), so computing a
    sub-range reproduces those U_k bit for bit — for the SU(2)-form, Lie–Trotter and general spin-one kernels."""
    w = {"C4": lambda: W.c4_long(duration=1e-3), "C2": lambda: W.c2_neural(duration=1e-3),
         "G1": lambda: W.g1_su3(batch=3, duration=1e-3)}[which]()
    sim = ss.Simulator(w.spin, w.method, w.expo, w.tau, w.frame, "fp64", w.field)
    sweep = torch.from_numpy(w.sweep).cuda()
    full = sim.compute_unitaries(sweep, w.t0, w.t1, w.dt_int, w.dt_out)
    part = sim.compute_unitaries(sweep, w.t0, w.t1, w.dt_int, w.dt_out, k_begin=333, k_count=100)
    assert torch.equal(full[:, 333:433], part)


def test_unitarity_and_norm(ss):
    w = W.c2_neural(duration=20e-3).with_(psi0=W.random_states(1, 3, seed=31))
    st, U = gpu_run(ss, w)
    UhU = np.conj(np.transpose(U[0], (0, 2, 1))) @ U[0]
    assert np.abs(UhU - np.eye(3)).max() < 1e-12
    assert np.abs(np.linalg.norm(st[0], axis=1) - 1).max() < 1e-12


@pytest.mark.parametrize("d", [2, 3])
@pytest.mark.parametrize("B,K", [(3, 1031), (4100, 9)])        # tiled scan and per-sweep chain kernel
@pytest.mark.parametrize("want_states", [True, False])
def test_scan_with_fused_spin_projection(ss, orc, d, B, K, want_states):
    """⟨J⟩ fused into the state write-out equals the oracle's projection of its own chain."""
    U = _random_unitaries(B, K, d, seed=B + K + d)
    psi0 = W.random_states(B, d, seed=32)
    ref_states = orc.chain(U, psi0)
    ref_spin = orc.spin_projection("half" if d == 2 else "one", ref_states)
    st, spin = ss.scan_states_spin(torch.from_numpy(U).cuda(), torch.from_numpy(psi0).cuda(), want_states=want_states)
    assert np.abs(spin.cpu().numpy() - ref_spin).max() < 1e-12
    if want_states:
        assert np.abs(st.cpu().numpy() - ref_states).max() < 1e-12
    else:
        assert st is None


def test_cuda_graph_capture_replay(ss):
    """ss_evaluate (validation off) is stream-ordered and capturable: a CUDA graph replay reproduces the direct call
    bit for bit (the way a sweep loop would amortise launch overhead)."""
    w = W.c2_neural(duration=2e-3)
    sim = ss.Simulator(w.spin, w.method, w.expo, w.tau, w.frame, "fp64", w.field)
    sweep = torch.from_numpy(w.sweep).cuda()
    psi0 = torch.from_numpy(w.psi0).cuda()
    ref = sim.evaluate(sweep, w.t0, w.t1, w.dt_int, w.dt_out, psi0)       # also warms up first-call attributes
    sim.set_validation(False)
    K = w.K
    states = torch.empty((1, K + 1, 3), dtype=torch.complex128, device="cuda")
    U = torch.empty((1, K, 3, 3), dtype=torch.complex128, device="cuda")
    ws = torch.empty(sim.workspace_bytes(1, K, False), dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        sim.evaluate(sweep, w.t0, w.t1, w.dt_int, w.dt_out, psi0, workspace=ws, out_states=states, out_unitaries=U)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        sim.evaluate(sweep, w.t0, w.t1, w.dt_int, w.dt_out, psi0, workspace=ws, out_states=states, out_unitaries=U)
    states.zero_()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(states, ref.state) and torch.equal(U, ref.time_evolution)


@pytest.mark.parametrize("spin,expo", [("half", "analytic"), ("one", "analytic"), ("one", "lie_trotter")])
def test_pulse_window_edges_parity(ss, orc, spin, expo):
    """The specialised pulse-free step body (DESIGN.md §5 item 12) is taken only for intervals that provably miss the
    sinp cycle: put the window's start and end exactly on interval boundaries, on fine-step boundaries and between
    the two Gauss points of a step, over many sweeps, and compare element by element with the oracle."""
    dt_out, L = 1e-6, 8
    dt = dt_out / L
    ws = 2 * np.pi / (5 * dt_out)                         # one sinp cycle = 5 intervals
    t_ps = [10 * dt_out, 10 * dt_out + dt, 10 * dt_out + 0.5 * dt, 10 * dt_out + 0.2113 * dt,
            10 * dt_out - 1e-15, 13 * dt_out + 3 * dt, 12.5 * dt_out]
    rows = [W.neural_params(omega_bias=2 * np.pi * 7e5, omega_dress=2 * np.pi * 20e3, omega_pulse=2 * np.pi * 30e3,
                            omega_sig=ws, t_p=tp, omega_q=(2 * np.pi * 72 if expo == "lie_trotter" else 0.0))
            for tp in t_ps]
    d = 2 if spin == "half" else 3
    w = W.Workload("pulse_edges", spin, "cf4", expo, 24, True, "neural", 0.0, 24 * dt_out, dt, dt_out,
                   np.stack(rows), W.random_states(len(rows), d, seed=41))
    assert_parity(ss, orc, w)


# ---- degenerate and minimal problems -------------------------------------------------------------------------------
@pytest.mark.parametrize("spin,expo,field,nc", [("half", "analytic", "constant", 4), ("one", "lie_trotter", "constant", 4),
                                                ("one", "analytic", "constant", 4),
                                                ("one", "lie_trotter_su3", "su3_constant", 8)])
@pytest.mark.parametrize("frame", [True, False])
def test_zero_field_is_identity(ss, spin, expo, field, nc, frame):
    """H ≡ 0: every exponential, product and frame factor is exactly the identity, so ψ_k = ψ0 bit for bit and every
    U_k is exactly I (any stray term in a residual formula would show)."""
    d = 2 if spin == "half" else 3
    w = W.Workload("zero", spin, "cf4", expo, 24, frame, field, 0.0, 7e-6, 0.5e-6, 1e-6, np.zeros((3, nc)),
                   W.random_states(3, d, seed=61))
    st, U = gpu_run(ss, w)
    assert np.array_equal(U, np.broadcast_to(np.eye(d, dtype=complex), U.shape))
    assert np.array_equal(st, np.broadcast_to(w.psi0[:, None, :], st.shape))


@pytest.mark.parametrize("spin,expo", [("half", "analytic"), ("one", "lie_trotter"), ("one", "analytic"),
                                       ("one", "lie_trotter_su3")])
@pytest.mark.parametrize("K,L", [(1, 1), (1, 1000), (3, 1)])
def test_minimal_grids_parity(ss, orc, spin, expo, K, L):
    """Smallest grids (one interval, one fine step; one interval of 1000 steps — the widest sub-interval split)
    through every exponentiator, against the oracle."""
    d = 2 if spin == "half" else 3
    p = W.neural_params(t_p=0.0, omega_q=(0.0 if expo == "analytic" else W.OMEGA_Q))
    w = W.Workload("min", spin, "cf4", expo, 24, True, "neural", 0.0, K * 1e-6, 1e-6 / L, 1e-6, p[None, :],
                   W.random_states(1, d, seed=62))
    assert_parity(ss, orc, w)
