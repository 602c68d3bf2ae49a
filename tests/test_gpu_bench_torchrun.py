"""bench.py under torchrun, the way the driver's SCALE run launches it (`python -m torch.distributed.run
--nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N`), with the two ranks sharing the one test GPU over
gloo (NCCL refuses two ranks per device): the sweep-sharded C3 line, the time-partitioned C4 line and the reference
arm each print exactly one JSON line, from rank 0, with the whole job's accounting.  A code-path check, not a timing."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def torchrun(args, timeout=900):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"), "--gpus", "2", *args]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


SHARED = ["--share-gpu", "--dist-backend", "gloo", "--steps", "1", "--warmup", "3", "--no-e2e", "--no-cpu-baseline",
          "--no-probe"]


def test_c3_sweep_sharding_two_ranks():
    d = torchrun(SHARED + ["--batch", "256"])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0
    assert d["config"]["global_batch"] == 256 and d["config"]["parallelism"] == "sweep-shard x2"
    assert d["fine_steps_per_step"] == 256 * 10000 * 10


def test_c4_time_partition_two_ranks():
    d = torchrun(SHARED + ["--workload", "C4"])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["config"]["k_per_rank"] == 500000
    assert "time-partition x2" in d["config"]["parallelism"]


def test_reference_arm_two_ranks():
    d = torchrun(["--impl", "reference", "--steps", "1", "--warmup", "0", "--ref-step-seconds", "1"])
    assert d["impl"] == "reference" and d["value"] > 0
