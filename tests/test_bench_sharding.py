"""bench.py's own multi-rank bookkeeping on CPU (gloo, world size 2): the sweep shards of the strong- and weak-scaling
C3 lines (BASELINE configs[2]: 8192 sweeps sharded across the GPUs), the one-GPU shard emulation, the MAX-over-ranks
timing reduction and C4's time partition (BASELINE configs[3]) — the code the driver's SCALE run executes, minus the
kernels."""
import argparse
import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp


def _args(**kw):
    a = dict(workload="C3", batch=8192, scaling="strong", emulate_ranks=1, expo=None)
    a.update(kw)
    return argparse.Namespace(**a)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        from paper_2204_05586_b200.distributed import partition_bounds
        strong = bench.shard_of(_args(), rank, world)
        weak = bench.shard_of(_args(scaling="weak"), rank, world)
        # MAX over ranks: every rank reports its own times, all receive the largest
        mx = bench.reduce_max([1.0 + rank, 10.0 - rank], None, world)
        kb, kc = partition_bounds(1_000_000, world, rank)
        q.put((rank, strong[:2], strong[2].batch, weak[:2], weak[2].batch, mx, kb, kc,
               strong[2].sweep[strong[0]:strong[1]].sum()))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_bench_sharding_gloo_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
        assert p.exitcode == 0
    res = sorted(q.get() for _ in range(world))
    # strong scaling: the 8192 sweeps of configs[2] split into two contiguous blocks of 4096, whole job = 8192
    assert [r[1] for r in res] == [(0, 4096), (4096, 8192)] and all(r[2] == 8192 for r in res)
    # weak scaling: 8192 sweeps per rank, the job's workload holds 16384
    assert [r[3] for r in res] == [(0, 8192), (8192, 16384)] and all(r[4] == 16384 for r in res)
    assert all(r[5] == [2.0, 10.0] for r in res)
    # C4: 1e6 intervals in two halves
    assert [(r[6], r[7]) for r in res] == [(0, 500_000), (500_000, 500_000)]
    # the two shards are different sweeps of the one grid
    assert res[0][8] != res[1][8]


def test_bench_emulated_shard_matches_rank0():
    """--emulate-ranks N on one process times exactly rank 0's block of the N-rank strong-scaling job."""
    import bench
    for n in (2, 4, 8):
        lo, hi, full = bench.shard_of(_args(emulate_ranks=n), 0, 1)
        assert (lo, hi) == (0, 8192 // n) and full.batch == 8192
        assert np.array_equal(full.sweep[lo:hi], bench.shard_of(_args(), 0, n)[2].sweep[:8192 // n])
