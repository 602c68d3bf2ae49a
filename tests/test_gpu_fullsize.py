"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times, on outputs the oracle can
compute one by one (sampled sweeps / sampled intervals / prefixes), plus properties that hold at any size.
Tolerances: 1e-10 max abs amplitude error (FP64), 1e-4 (FP32 mode) — BASELINE.json north_star."""
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


def run_gpu(ss, w, precision="fp64", want_unitaries=True):
    sim = ss.Simulator(w.spin, w.method, w.expo, w.tau, w.frame, precision, w.field)
    res = sim.evaluate(torch.from_numpy(w.sweep).cuda(), w.t0, w.t1, w.dt_int, w.dt_out,
                       torch.from_numpy(w.psi0).cuda(), want_unitaries=want_unitaries)
    torch.cuda.synchronize()
    return sim, res


def oracle_sweeps(orc, w, idx, **kw):
    return orc.evaluate(w.spin, w.method, w.expo, w.tau, w.frame, w.field, sweep=w.sweep[idx], t0=w.t0, t1=w.t1,
                        dt_int=w.dt_int, dt_out=w.dt_out, psi0=w.psi0[idx], **kw)


def unitarity_and_norm(res):
    U = res.time_evolution
    d = U.shape[-1]
    eye = torch.eye(d, dtype=U.dtype, device=U.device)
    dev = 0.0
    for chunk in torch.split(U, 256):
        dev = max(dev, (chunk.conj().transpose(-1, -2) @ chunk - eye).abs().max().item())
    norm = (res.state.abs().pow(2).sum(-1).sqrt() - 1).abs().max().item()
    return dev, norm


def test_c3_full_8192_sweeps(ss, orc):
    """C3 exactly as bench.py runs it: 8192 spin-one sweeps × 10 ms (8.19e8 fine steps)."""
    w = W.c3_batched()
    _, res = run_gpu(ss, w)
    idx = np.array([0, 1, 63, 127, 2047, 4096, 6000, 8191])
    st_o, U_o = oracle_sweeps(orc, w, idx)
    st_g = res.state[torch.from_numpy(idx).cuda()].cpu().numpy()
    U_g = res.time_evolution[torch.from_numpy(idx).cuda()].cpu().numpy()
    assert np.abs(U_g - U_o).max() <= 1e-10
    assert np.abs(st_g - st_o).max() <= 1e-10
    dev, norm = unitarity_and_norm(res)
    assert dev < 1e-12                      # every one of the 8.2e7 interval operators
    assert norm < 1e-11                     # K = 1e4 intervals: chain drift ~3e-17 per interval


@pytest.mark.parametrize("dt_int", [100e-9, 10e-9])
def test_c2_full_100ms(ss, orc, dt_int):
    """C2: the paper's spin-one benchmark, 100 ms, δt = 100 ns (1e6 steps) and 10 ns (1e7 steps), K = 1e5."""
    w = W.c2_neural(dt_int=dt_int)
    _, res = run_gpu(ss, w)
    st_o, U_o = oracle_sweeps(orc, w, [0])
    assert np.abs(res.time_evolution.cpu().numpy() - U_o).max() <= 1e-10
    assert np.abs(res.state.cpu().numpy() - st_o).max() <= 1e-10


@pytest.mark.parametrize("expo", ["lie_trotter", "analytic"])
def test_c5_full_fp64_and_fp32(ss, orc, expo):
    """C5: Eq. neural_pulse as printed (ω_q = 0), 100 ms, δt = 100 ns; FP64 ≤ 1e-10 and FP32 ≤ 1e-4 vs the oracle."""
    w = W.c5_matrix(expo)
    st_o, _ = oracle_sweeps(orc, w, [0], want_unitaries=False)
    _, r64 = run_gpu(ss, w, want_unitaries=False)
    assert np.abs(r64.state.cpu().numpy() - st_o).max() <= 1e-10
    _, r32 = run_gpu(ss, w, precision="fp32", want_unitaries=False)
    assert np.abs(r32.state.cpu().numpy() - st_o).max() <= 1e-4


@pytest.mark.parametrize("expo,precision,want_unitaries", [("lie_trotter", "fp64", True),
                                                           ("analytic", "fp64", False),
                                                           ("analytic", "fp32", False),
                                                           ("lie_trotter", "fp32", False)])
def test_c5_throughput_batch_sampled(ss, orc, expo, precision, want_unitaries):
    """C5's throughput workload (100 sweeps × 1e5 intervals) in the launch configuration bench.py times — the fused
    path (run products in the interval kernel, coarse scan, run chain), compact operators when U is not requested —
    sampled sweeps against the oracle at the precision's bar."""
    w = W.c5_matrix(expo, batch=100)
    _, res = run_gpu(ss, w, precision=precision, want_unitaries=want_unitaries)
    idx = np.array([0, 49, 99])
    st_o, U_o = oracle_sweeps(orc, w, idx, want_unitaries=want_unitaries)
    tol = 1e-10 if precision == "fp64" else 1e-4
    assert np.abs(res.state[torch.from_numpy(idx).cuda()].cpu().numpy() - st_o).max() <= tol


def test_c4_full_1s_at_1ns(ss, orc):
    """C4: one spin-half simulation, 1 s at δt = 1 ns (1e9 fine steps, K = 1e6, L = 1000).  Sampled intervals are
    compared operator by operator; the state is compared over the oracle-feasible prefix; norm over all K."""
    w = W.c4_long()
    sim, res = run_gpu(ss, w)
    ks = np.array([0, 1, 2, 233000, 233500, 500000, 999998, 999999])   # incl. the pulse at t_p = 233 ms
    U_g = res.time_evolution[0, torch.from_numpy(ks).cuda()].cpu().numpy()
    for k, Ug in zip(ks, U_g):
        _, U_o = orc.evaluate(w.spin, w.method, w.expo, w.tau, w.frame, w.field, sweep=w.sweep, t0=w.t0, t1=w.t1,
                              dt_int=w.dt_int, dt_out=w.dt_out, psi0=w.psi0, k_begin=int(k), k_end=int(k) + 1)
        assert np.abs(Ug - U_o[0, 0]).max() <= 1e-12
    # prefix [0, 5 ms] chained by the oracle from the GPU-identical time grid
    pre = w.with_(t1=5e-3)
    st_o, _ = oracle_sweeps(orc, pre, [0], want_unitaries=False)
    assert np.abs(res.state[0, : pre.K + 1].cpu().numpy() - st_o[0]).max() <= 1e-10
    dev, norm = unitarity_and_norm(res)
    assert dev < 1e-12
    assert norm < 1e-9          # 1e6 intervals: report-level drift bound (~3e-17/interval)


def test_c4_virtual_time_partition_matches_single_gpu(ss):
    """The time-partition code path (aggregates → carry → local scan) over 8 virtual parts reproduces the
    single-GPU states (association differences only)."""
    from paper_2204_05586_b200.distributed import evaluate_virtual_partition
    w = W.c4_long(duration=0.1)
    sim, res = run_gpu(ss, w, want_unitaries=False)
    st = evaluate_virtual_partition(sim, torch.from_numpy(w.sweep).cuda(), w.t0, w.t1, w.dt_int, w.dt_out,
                                    torch.from_numpy(w.psi0).cuda(), n_parts=8)
    assert st.shape == res.state.shape
    assert (st - res.state).abs().max().item() < 1e-12


def test_c1_full_both_drives(ss, orc):
    for field in ("rabi_circular", "rabi_linear"):
        w = W.c1_rabi(field)
        _, res = run_gpu(ss, w)
        st_o, U_o = oracle_sweeps(orc, w, [0])
        assert np.abs(res.state.cpu().numpy() - st_o).max() <= 1e-10
