"""The NCCL branch of the time partition's one exchange (distributed.gather_aggregates → all_gather_into_tensor) on
the B200: the round-end GPU box has one GPU, and NCCL refuses two ranks on one device, so this runs the real NCCL
collective at world size 1 in a child process (its own process group) — the rank-0 slice of an all-gather over real
C4 aggregates from the library — and checks it returns the aggregates unchanged.  The multi-rank bookkeeping around
it is covered with gloo (tests/test_distributed.py, tests/test_gpu_distributed.py)."""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import os, sys, torch, numpy as np
import torch.distributed as dist
sys.path.insert(0, os.environ["SS_ROOT"])
import paper_2204_05586_b200 as ss, workloads as W
from paper_2204_05586_b200.distributed import gather_aggregates, time_partitioned, library_steps
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
assert dist.get_backend() == "nccl"
w = W.c4_long(duration=2e-3)
sim = ss.Simulator(w.spin, w.method, w.expo, w.tau, w.frame, "fp64", w.field)
sweep = torch.from_numpy(w.sweep).cuda()
U = sim.compute_unitaries(sweep, w.t0, w.t1, w.dt_int, w.dt_out)
A = ss.chain_aggregate(U)
G = gather_aggregates(A)                                      # NCCL all_gather_into_tensor
torch.cuda.synchronize()
assert G.shape == (1, *A.shape) and torch.equal(G[0], A), "NCCL gather changed the aggregate"
# the partition driver with the NCCL gather wired in, one part: equals the single-call states
steps = library_steps(sim, sweep, w.t0, w.t1, w.dt_int, w.dt_out)
psi0 = torch.from_numpy(w.psi0).cuda()
kb, st = time_partitioned(steps, w.K, psi0, 0, 1, gather_aggregates)
ref = ss.scan_states(U, psi0)
assert kb == 0 and torch.equal(st, ref)
dist.destroy_process_group()
print("nccl ok", torch.cuda.nccl.version())
"""


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_nccl_gather_aggregates_world1():
    env = dict(os.environ, SS_ROOT=ROOT, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), NCCL_DEBUG="INFO")
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-4000:])
    assert "nccl ok" in r.stdout
    assert "NCCL INFO" in r.stdout + r.stderr         # the collective really initialised NCCL
