"""Multi-rank paths on real kernels: two processes sharing the one available GPU, exchanging over gloo (NCCL refuses
two ranks on one device).  Checks the time-partitioned simulation end to end (global-k operators, aggregate
all-gather, carry composition, scan from the carry) against the single-process run."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import workloads as W

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_2204_05586_b200 as ss
        from paper_2204_05586_b200.distributed import evaluate_time_partitioned
        w = W.c4_long(duration=10e-3)
        sim = ss.Simulator(w.spin, w.method, w.expo, w.tau, w.frame, "fp64", w.field)
        kb, st = evaluate_time_partitioned(sim, torch.from_numpy(w.sweep).cuda(), w.t0, w.t1, w.dt_int, w.dt_out,
                                           torch.from_numpy(w.psi0).cuda())
        torch.cuda.synchronize()
        q.put((rank, kb, st.cpu().numpy()))
    finally:
        dist.destroy_process_group()


def test_time_partition_two_ranks_one_gpu():
    import paper_2204_05586_b200 as ss
    w = W.c4_long(duration=10e-3)
    sim = ss.Simulator(w.spin, w.method, w.expo, w.tau, w.frame, "fp64", w.field)
    ref = sim.evaluate(torch.from_numpy(w.sweep).cuda(), w.t0, w.t1, w.dt_int, w.dt_out,
                       torch.from_numpy(w.psi0).cuda(), want_unitaries=False).state.cpu().numpy()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=300) for _ in range(2)), key=lambda x: x[0])
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert res[0][1] == 0 and res[1][1] == w.K // 2
    for _, kb, st in res:
        assert np.abs(st - ref[:, kb:kb + st.shape[1]]).max() < 1e-12


def _shard_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_2204_05586_b200 as ss
        from paper_2204_05586_b200.distributed import shard_sweeps
        w = W.c3_batched(batch=96, duration=0.3e-3)
        sl = shard_sweeps(w.batch, rank, world)
        sim = ss.Simulator(w.spin, w.method, w.expo, w.tau, w.frame, "fp64", w.field)
        res = sim.evaluate(torch.from_numpy(np.ascontiguousarray(w.sweep[sl])).cuda(), w.t0, w.t1, w.dt_int, w.dt_out,
                           torch.from_numpy(np.ascontiguousarray(w.psi0[sl])).cuda(), want_unitaries=False)
        torch.cuda.synchronize()
        q.put((rank, sl.start, res.state.cpu().numpy()))
    finally:
        dist.destroy_process_group()


def test_sweep_sharding_three_ranks_bitwise():
    """C3-style sweep sharding: each rank evaluates its contiguous block of sweeps; the per-sweep states
    are bit-identical to the single-process run (same kernels, same split S here, same per-sweep decomposition)."""
    import paper_2204_05586_b200 as ss
    w = W.c3_batched(batch=96, duration=0.3e-3)
    sim = ss.Simulator(w.spin, w.method, w.expo, w.tau, w.frame, "fp64", w.field)
    ref = sim.evaluate(torch.from_numpy(w.sweep).cuda(), w.t0, w.t1, w.dt_int, w.dt_out,
                       torch.from_numpy(w.psi0).cuda(), want_unitaries=False).state.cpu().numpy()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=300) for _ in range(3)), key=lambda x: x[0])
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    got = np.concatenate([st for _, _, st in res], axis=0)
    assert got.shape == ref.shape
    assert np.array_equal(got, ref)
