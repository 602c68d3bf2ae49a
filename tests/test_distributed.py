"""Multi-process host logic of the multi-GPU layer on CPU (gloo, world size 2): partition bounds, the aggregate
exchange (ordering by rank), the carry composition order and the sweep sharding.  The compute steps are injected as
plain numpy/torch functions here — this checks bookkeeping only; the kernels themselves are covered by -m gpu."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2204_05586_b200.distributed import (PartitionSteps, gather_aggregates, partition_bounds, shard_sweeps,
                                               time_partitioned)


def test_partition_bounds_cover_exactly():
    for n in (1, 7, 8, 1000, 1000003):
        for world in (1, 2, 3, 4, 8):
            spans = [partition_bounds(n, world, r) for r in range(world)]
            assert spans[0][0] == 0
            for (b0, c0), (b1, _) in zip(spans, spans[1:]):
                assert b0 + c0 == b1
            assert sum(c for _, c in spans) == n
            assert max(c for _, c in spans) - min(c for _, c in spans) <= 1
    with pytest.raises(ValueError):
        partition_bounds(10, 2, 2)


def test_shard_sweeps():
    for B in (8192, 100, 3):
        for world in (1, 2, 4, 8):
            idx = np.concatenate([np.arange(B)[shard_sweeps(B, r, world)] for r in range(world)])
            assert np.array_equal(idx, np.arange(B))


def _unitaries(B, K, d, seed):
    rng = np.random.default_rng(seed)
    z = rng.standard_normal((B, K, d, d)) + 1j * rng.standard_normal((B, K, d, d))
    q, r = np.linalg.qr(z)
    return q * (np.diagonal(r, axis1=-2, axis2=-1) / np.abs(np.diagonal(r, axis1=-2, axis2=-1)))[..., None, :]


def _chain(U, psi0):
    B, K, d, _ = U.shape
    out = np.zeros((B, K + 1, d), complex)
    out[:, 0] = psi0
    for k in range(K):
        out[:, k + 1] = np.einsum("bij,bj->bi", U[:, k], out[:, k])
    return out


def _numpy_steps(U_full):
    def aggregate(U):
        U = U.numpy()
        A = np.broadcast_to(np.eye(U.shape[-1], dtype=complex), (U.shape[0],) + U.shape[2:]).copy()
        for k in range(U.shape[1]):
            A = np.einsum("bij,bjk->bik", U[:, k], A)
        return torch.from_numpy(A)

    def compose(A_all, psi0, part):
        psi = psi0.numpy().copy()
        for g in range(part):
            psi = np.einsum("bij,bj->bi", A_all[g].numpy(), psi)
        return torch.from_numpy(psi)

    return PartitionSteps(
        compute_unitaries=lambda kb, kc: torch.from_numpy(np.ascontiguousarray(U_full[:, kb:kb + kc])),
        chain_aggregate=aggregate,
        compose_carry=compose,
        scan_states=lambda U, carry: torch.from_numpy(_chain(U.numpy(), carry.numpy())),
    )


def _worker(rank, world, port, B, K, d, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        U = _unitaries(B, K, d, seed=5)
        psi0 = np.ones((B, d), complex) / np.sqrt(d)
        kb, states = time_partitioned(_numpy_steps(U), K, torch.from_numpy(psi0), rank, world,
                                      lambda A: gather_aggregates(A))
        ref = _chain(U, psi0)
        err = float(np.abs(states.numpy() - ref[:, kb:kb + states.shape[1]]).max())
        # every rank must hold the same carries: gather each rank's first state
        first = torch.view_as_real(states[:, 0].contiguous()).reshape(-1)
        parts = [torch.empty_like(first) for _ in range(world)]
        dist.all_gather(parts, first)
        q.put((rank, kb, states.shape[1] - 1, err))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("d", [2, 3])
def test_time_partition_gloo_world2(d):
    world, B, K = 2, 3, 37
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, B, K, d, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get() for _ in range(world))
    assert [r[1] for r in res] == [0, 19]           # bounds: 19 + 18 intervals
    assert sum(r[2] for r in res) == K
    for _, _, _, err in res:
        assert err < 1e-12
