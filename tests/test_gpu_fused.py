"""Fused run aggregates (DESIGN.md §5 item 16): for long problems each interval-kernel thread computes ipt consecutive
intervals and multiplies their U_k into a run aggregate, a coarse scan turns the aggregates into run start states, and
one chain thread per run writes the states (ss_evaluate below the chain kernel's batch size, S = 1).

* The whole path against the long-double oracle (≤ 1e-10), with ipt forced to 4, 8, 32 (SPINSIM_FUSED_IPT; runs
  longer than the operator type allows — dense 3×3: 8, dense 2×2: 16 — fall back to the unfused path), both operator
  formats (compact SU(2) without U, dense with U), both spins and all three spin-one exponentiators; one problem large
  enough for the heuristic to fuse; K not divisible by ipt (unfused).
* Against the unfused path (SPINSIM_FUSED=0): U_k bit for bit (the same per-interval arithmetic, only the thread →
  interval map differs), states to rounding (a different product association).
* The coarse scan through every state-scan kernel (SPINSIM_SCAN_PATH), and the launch count that shows the fused
  path ran.
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


def _shape(name):
    """Shapes whose split heuristic (DESIGN.md §5 item 8) takes S = 1: L = 5 admits no split."""
    if name == "half":               # 3 spin-half sweeps, K = 992
        return W.c4_long(duration=992e-6, dt_int=200e-9).with_(
            sweep=np.repeat(W.c4_long().sweep, 3, 0) * np.array([[1.0], [1.01], [0.99]]), psi0=W.random_states(3, 2, 61))
    if name == "one_lt":             # 2 spin-one Lie–Trotter sweeps, K = 800
        return W.c5_matrix("lie_trotter", batch=2).with_(t1=800e-6, dt_int=200e-9, psi0=W.random_states(2, 3, 62))
    if name == "one_an":             # 5 analytic spin-one sweeps, K = 480
        return W.c5_matrix("analytic", batch=5).with_(t1=480e-6, dt_int=200e-9, psi0=W.random_states(5, 3, 63))
    if name == "one_su3":            # 3 general spin-one sweeps, K = 416
        w = W.g1_su3(batch=3, duration=416e-6)
        return w.with_(dt_int=200e-9, psi0=W.random_states(3, 3, 64))
    raise KeyError(name)


def _eval(ss, w, want_unitaries, monkeypatch, fused, ipt=None):
    monkeypatch.setenv("SPINSIM_FUSED", "1" if fused else "0")
    if ipt is None:
        monkeypatch.delenv("SPINSIM_FUSED_IPT", raising=False)
    else:
        monkeypatch.setenv("SPINSIM_FUSED_IPT", str(ipt))
    sim = ss.Simulator(w.spin, w.method, w.expo, w.tau, w.frame, "fp64", w.field)
    n0 = ss.kernel_launches()
    res = sim.evaluate(torch.from_numpy(w.sweep).cuda(), w.t0, w.t1, w.dt_int, w.dt_out,
                       torch.from_numpy(w.psi0).cuda(), want_unitaries=want_unitaries)
    torch.cuda.synchronize()
    n = ss.kernel_launches() - n0
    U = res.time_evolution.cpu().numpy() if want_unitaries else None
    return res.state.cpu().numpy(), U, n


def _oracle(orc, w):
    return orc.evaluate(w.spin, w.method, w.expo, w.tau, w.frame, w.field, sweep=w.sweep, t0=w.t0, t1=w.t1,
                        dt_int=w.dt_int, dt_out=w.dt_out, psi0=w.psi0)


@pytest.mark.parametrize("want_unitaries", [False, True])
@pytest.mark.parametrize("ipt", [4, 8, 32])
@pytest.mark.parametrize("name", ["half", "one_lt", "one_an", "one_su3"])
def test_fused_vs_oracle_and_unfused(ss, orc, monkeypatch, name, ipt, want_unitaries):
    w = _shape(name)
    assert w.L == 5 and w.K % 32 == 0, "shape must take S = 1 and split into whole runs"
    st, U, n_fused = _eval(ss, w, want_unitaries, monkeypatch, fused=True, ipt=ipt)
    st0, U0, n_plain = _eval(ss, w, want_unitaries, monkeypatch, fused=False)
    compact = not want_unitaries and (w.spin == "half" or w.expo == "analytic")
    max_ipt = 32 if compact else (16 if w.spin == "half" else 8)
    # validation + interval kernel + coarse scan (≥ 1 kernel) + run chain, against validation + interval + scan
    if ipt <= max_ipt:
        assert n_fused >= n_plain + 1, (n_fused, n_plain)
    else:
        assert n_fused == n_plain, (n_fused, n_plain)
    ref = _oracle(orc, w)
    assert np.abs(st - ref[0]).max() <= 1e-10, name
    assert np.abs(st - st0).max() <= max(1e-12, 6e-17 * w.K), name
    assert np.array_equal(st[:, 0], w.psi0)
    if want_unitaries:
        assert np.array_equal(U, U0), "fused launch changed the interval operators"
        assert np.abs(U - ref[1]).max() <= 1e-12


def test_fused_by_heuristic(ss, orc, monkeypatch):
    """One spin-half sweep of 5e6 intervals (L = 10): ≥ 16 waves at 4 intervals per thread, so ss_evaluate fuses
    without being told; states against the oracle and the unfused path."""
    w = W.c4_long(duration=5_000_000 * 1e-8, dt_int=1e-9, dt_out=1e-8)
    st, _, n_fused = _eval(ss, w, False, monkeypatch, fused=True)
    st0, _, n_plain = _eval(ss, w, False, monkeypatch, fused=False)
    # unfused, 160 MB of compact operators take the standalone two-pass scan (its own run-products kernel); fused,
    # the interval kernel wrote the run products: validation, interval kernel, coarse scan, run chain
    assert n_fused == 4 and n_plain == n_fused + 1, (n_fused, n_plain)
    ref = _oracle(orc, w.with_(t1=w.t0 + 20000 * w.dt_out))[0]          # the oracle on a prefix (20 000 intervals)
    assert np.abs(st[:, :20001] - ref).max() <= 1e-10
    assert np.abs(st - st0).max() <= 6e-17 * w.K
    assert abs(np.linalg.norm(st[0, -1]) - 1.0) < 1e-9


@pytest.mark.parametrize("path", ["coop", "scan2", "scan3", "twopass", "chain"])
def test_fused_coarse_scan_every_path(ss, orc, monkeypatch, path):
    """The coarse scan over the run aggregates through each state-scan kernel (the heuristic picks one by size)."""
    w = _shape("one_an").with_(t1=3000e-6)
    monkeypatch.setenv("SPINSIM_SCAN_PATH", path)
    ref = _oracle(orc, w)[0]
    for want_unitaries in (False, True):
        st, _, _ = _eval(ss, w, want_unitaries, monkeypatch, fused=True, ipt=4)
        assert np.abs(st - ref).max() <= 1e-10, (path, want_unitaries)


def test_fused_single_run_and_tiny(ss, orc, monkeypatch):
    """Degenerate sizes: K = 2·ipt (two runs, the smallest fused problem); K = 17, 15, 3 are not multiples of ipt and
    take the unfused path."""
    base = _shape("one_an")
    for K in (16, 17, 15, 3):
        w = base.with_(t1=K * 1e-6, sweep=base.sweep[:1], psi0=base.psi0[:1])
        st, _, _ = _eval(ss, w, False, monkeypatch, fused=True, ipt=8)
        assert np.abs(st - _oracle(orc, w)[0]).max() <= 1e-12, K


@pytest.mark.parametrize("name", ["one_an", "half"])
def test_fused_host_pipeline(ss, monkeypatch, name):
    """ss_evaluate_host runs each chunk through the same launch path (fused where the chunk allows): batch chunks and
    time chunks against the unfused device call, to rounding."""
    w = _shape(name)
    st0, _, _ = _eval(ss, w, False, monkeypatch, fused=False)
    monkeypatch.setenv("SPINSIM_FUSED", "1")
    monkeypatch.setenv("SPINSIM_FUSED_IPT", "8")
    sim = ss.Simulator(w.spin, w.method, w.expo, w.tau, w.frame, "fp64", w.field)
    for chunks in (0, 1, 2, 6):
        st_h, _ = sim.evaluate_host(w.sweep, w.t0, w.t1, w.dt_int, w.dt_out, w.psi0, want_unitaries=False,
                                    n_chunks=chunks)
        assert np.abs(st_h - st0).max() <= 1e-12, chunks


NEURAL_USER_SRC = r"""
__device__ void user_field(double t_k, double off, const double* p, double f[4]) {
  const double t = t_k + off;
  f[0] = 2.0 * p[2] * cos(p[1] * t);
  const double x = p[4] * ((t_k - p[5]) + off);
  f[2] = p[0] + ((x >= 0.0 && x <= 6.283185307179586) ? p[3] * sin(x) : 0.0);
  f[3] = p[6];
}
"""


@pytest.mark.parametrize("spin", ["half", "one"])
def test_fused_user_field(ss, orc, monkeypatch, spin):
    """The run-time compiled (NVRTC) interval kernel takes the fused mode too (its dynamic shared memory and mode
    branch): a user copy of Eq. neural_pulse against the oracle's built-in field, ipt forced."""
    w = _shape("half" if spin == "half" else "one_lt")
    monkeypatch.setenv("SPINSIM_FUSED", "1")
    monkeypatch.setenv("SPINSIM_FUSED_IPT", "8")
    sim = ss.Simulator(w.spin, w.method, w.expo, w.tau, w.frame, "fp64", "user", field_source=NEURAL_USER_SRC,
                       n_params=7)
    n0 = ss.kernel_launches()
    for want_unitaries in (False, True):
        res = sim.evaluate(torch.from_numpy(w.sweep).cuda(), w.t0, w.t1, w.dt_int, w.dt_out,
                           torch.from_numpy(w.psi0).cuda(), want_unitaries=want_unitaries)
        assert np.abs(res.state.cpu().numpy() - _oracle(orc, w)[0]).max() <= 1e-10
    assert ss.kernel_launches() - n0 >= 2 * 4                # validation, interval, coarse scan, run chain (each call)


@pytest.mark.parametrize("expo", ["lie_trotter", "analytic"])
def test_fused_fp32(ss, orc, monkeypatch, expo):
    """FP32 mode through the fused path (the FP64 run products and run chain over the FP32 kernel's operators)
    against the oracle at the FP32 bar, and against the unfused FP32 path to rounding."""
    w = _shape("one_lt" if expo == "lie_trotter" else "one_an")
    monkeypatch.setenv("SPINSIM_FUSED_IPT", "8")
    sim32 = ss.Simulator(w.spin, w.method, w.expo, w.tau, w.frame, "fp32", w.field)
    sweep, psi0 = torch.from_numpy(w.sweep).cuda(), torch.from_numpy(w.psi0).cuda()
    monkeypatch.setenv("SPINSIM_FUSED", "1")
    st32 = sim32.evaluate(sweep, w.t0, w.t1, w.dt_int, w.dt_out, psi0, want_unitaries=False).state.cpu().numpy()
    monkeypatch.setenv("SPINSIM_FUSED", "0")
    st32u = sim32.evaluate(sweep, w.t0, w.t1, w.dt_int, w.dt_out, psi0, want_unitaries=False).state.cpu().numpy()
    assert np.abs(st32 - _oracle(orc, w)[0]).max() <= 1e-4
    assert np.abs(st32 - st32u).max() <= 1e-12            # same FP32 operators, two FP64 product associations


@pytest.mark.parametrize("want_unitaries", [False, True])
def test_fused_cuda_graph_capture(ss, monkeypatch, want_unitaries):
    """The fused path (interval kernel with run products, coarse scan, run chain) is stream-ordered and capturable:
    a CUDA-graph replay reproduces the direct call bit for bit."""
    w = _shape("one_an")
    monkeypatch.setenv("SPINSIM_FUSED", "1")
    monkeypatch.setenv("SPINSIM_FUSED_IPT", "8")
    sim = ss.Simulator(w.spin, w.method, w.expo, w.tau, w.frame, "fp64", w.field)
    sweep, psi0 = torch.from_numpy(w.sweep).cuda(), torch.from_numpy(w.psi0).cuda()
    ref = sim.evaluate(sweep, w.t0, w.t1, w.dt_int, w.dt_out, psi0, want_unitaries=want_unitaries)
    sim.set_validation(False)
    B, K, D = w.batch, w.K, w.dim
    states = torch.empty((B, K + 1, D), dtype=torch.complex128, device="cuda")
    U = torch.empty((B, K, D, D), dtype=torch.complex128, device="cuda") if want_unitaries else None
    ws = torch.empty(sim.workspace_bytes(B, K, not want_unitaries), dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        sim.evaluate(sweep, w.t0, w.t1, w.dt_int, w.dt_out, psi0, want_unitaries=want_unitaries, workspace=ws,
                     out_states=states, out_unitaries=U)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        sim.evaluate(sweep, w.t0, w.t1, w.dt_int, w.dt_out, psi0, want_unitaries=want_unitaries, workspace=ws,
                     out_states=states, out_unitaries=U)
    states.zero_()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(states, ref.state)
    if want_unitaries:
        assert torch.equal(U, ref.time_evolution)
