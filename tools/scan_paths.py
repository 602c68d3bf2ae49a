"""Time every state-scan kernel (SPINSIM_SCAN_PATH override) on the paper-shaped scan problems, both operator formats.

    python tools/scan_paths.py > profiles/r02/<tag>/scan_paths.txt

Shapes (B sweeps × K intervals): C5 (100 × 1e5), the scan-stress sweep (1 × 1e8), one rank's shard of C3 at 8 GPUs
(1024 × 1e4), at 4 GPUs (2048 × 1e4) and at 2 GPUs (4096 × 1e4), C2 (1 × 1e5), C3 (8192 × 1e4).  Operators are random (unit quaternions →
SU(2) elements; dense = the same matrices written out, D¹ for dim 3) generated on the device; each kernel is timed
with CUDA events over 3 repetitions after a warm-up, and reported as algorithmic HBM bytes / time against 6534.8 GB/s.
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_05586_b200 as ss  # noqa: E402

HBM = 6534.8e9
PATHS = ["coop", "chain", "scan2", "scan3", "twopass"]


def random_ops(B, K, d, compact, gen):
    q = torch.randn((B, K, 4), dtype=torch.float64, device="cuda", generator=gen)
    q /= q.norm(dim=-1, keepdim=True)
    a = torch.complex(q[..., 0], q[..., 1])
    b = torch.complex(q[..., 2], q[..., 3])
    if compact:
        return torch.stack([a, b], -1).contiguous()
    if d == 2:
        return torch.stack([torch.stack([a, b], -1), torch.stack([-b.conj(), a.conj()], -1)], -2).contiguous()
    s2 = 2.0 ** 0.5
    return torch.stack([torch.stack([a * a, s2 * a * b, b * b], -1),
                        torch.stack([-s2 * a * b.conj(), a.abs() ** 2 - b.abs() ** 2 + 0j, s2 * a.conj() * b], -1),
                        torch.stack([b.conj() ** 2, -s2 * a.conj() * b.conj(), a.conj() ** 2], -1)], -2).contiguous()


def time_path(path, ops, psi0, d, compact, states, ws):
    os.environ["SPINSIM_SCAN_PATH"] = path
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    try:
        for rep in range(4):
            if rep == 1:
                ev[0].record()
            if compact:
                ss.scan_states_su2(ops, psi0, d, workspace=ws)
            else:
                ss.scan_states(ops, psi0, out=states, workspace=ws)
        ev[1].record()
        torch.cuda.synchronize()
    except Exception as exc:          # e.g. coop not eligible on this shape
        return None, str(exc).splitlines()[0][:60]
    finally:
        del os.environ["SPINSIM_SCAN_PATH"]
    return ev[0].elapsed_time(ev[1]) / 3, ""


def main():
    gen = torch.Generator(device="cuda")
    gen.manual_seed(7)
    shapes = [("C5", 100, 100000, 3), ("scan-stress", 1, 100000000, 2), ("C3 shard/8", 1024, 10000, 3),
              ("C3 shard/4", 2048, 10000, 3), ("C3 shard/2", 4096, 10000, 3), ("C2", 1, 100000, 3), ("C3", 8192, 10000, 3)]
    print(f"{'shape':12s} {'B':>5s} {'K':>10s} {'d':>2s} {'ops':7s} " + " ".join(f"{p:>17s}" for p in PATHS))
    for name, B, K, d in shapes:
        for compact in (True, False):
            nb = B * K * ((2 if compact else d * d) + d) * 16
            if nb > 40e9:
                continue
            ops = random_ops(B, K, d, compact, gen)
            psi0 = torch.zeros((B, d), dtype=torch.complex128, device="cuda")
            psi0[:, 0] = 1.0
            states = torch.empty((B, K + 1, d), dtype=torch.complex128, device="cuda")
            ws = torch.empty(int(ss._lib.load().ss_scan_workspace_bytes(d, B, K)), dtype=torch.uint8, device="cuda")
            cells = []
            for p in PATHS:
                if (p == "chain" and B < 1024) or (p == "coop" and (ops.numel() * 16 > 64 * 2 ** 20 or B > 512)):
                    cells.append(f"{'-':>17s}")       # not eligible (coop) / one sequential thread per sweep (chain)
                    continue
                ms, err = time_path(p, ops, psi0, d, compact, states, ws)
                cells.append(f"{ms:8.3f}ms {nb / (ms * 1e-3) / HBM:5.2f}" if ms else f"{'n/a':>17s}")
            print(f"{name:12s} {B:5d} {K:10d} {d:2d} {'su2' if compact else 'dense':7s} " + " ".join(cells),
                  flush=True)
            del ops, states, ws
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
