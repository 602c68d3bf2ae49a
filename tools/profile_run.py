"""Minimal launcher for ncu captures: one warm-up pass then `--reps` passes of the hot path (interval kernel +
scan) on a chosen workload, so `ncu -k regex:... -s 1 -c 1` lands on a warm launch.

    ncu --set full --clock-control none --import-source on -k regex:interval_kernel -s 1 -c 1 \
        -o gpurun_out/prof_interval python tools/profile_run.py --workload C3
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_05586_b200 as ss  # noqa: E402
import workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C3")
    ap.add_argument("--batch", type=int, default=8192)
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--precision", default="fp64")
    ap.add_argument("--duration", type=float, default=None)
    ap.add_argument("--expo", default=None, help="C5: analytic or lie_trotter")
    ap.add_argument("--evaluate", action="store_true",
                    help="the ss_evaluate path without U (compact SU(2) operators on the SU(2)-form paths)")
    args = ap.parse_args()
    w = {"C3": lambda: W.c3_batched(batch=args.batch), "C2": lambda: W.c2_neural(),
         "C4": lambda: W.c4_long(), "C5": lambda: W.c5_matrix(args.expo or "lie_trotter", batch=100),
         "C4S": lambda: W.c4_long(dt_int=1e-9, dt_out=10e-9, duration=1.0),
         "G1": lambda: W.g1_su3(batch=args.batch)}[args.workload]()
    if args.duration:
        w = w.with_(t1=w.t0 + args.duration)
    sim = ss.Simulator(w.spin, w.method, w.expo, w.tau, w.frame, args.precision, w.field)
    sweep = torch.from_numpy(w.sweep).cuda()
    psi0 = torch.from_numpy(w.psi0).cuda()
    st = torch.empty((w.batch, w.K + 1, w.dim), dtype=torch.complex128, device="cuda")
    if args.evaluate:
        ws = torch.empty(sim.workspace_bytes(w.batch, w.K, True), dtype=torch.uint8, device="cuda")
        sim.set_validation(False)
        for _ in range(1 + args.reps):
            sim.evaluate(sweep, w.t0, w.t1, w.dt_int, w.dt_out, psi0, want_unitaries=False, workspace=ws,
                         out_states=st)
        torch.cuda.synchronize()
        print("ok", w.name, w.batch, w.K, w.L, float(np.abs(st[0, -1].cpu().numpy()).sum()))
        return
    U = torch.empty((w.batch, w.K, w.dim, w.dim), dtype=torch.complex128, device="cuda")
    for _ in range(1 + args.reps):
        sim.compute_unitaries(sweep, w.t0, w.t1, w.dt_int, w.dt_out, out=U)
        ss.scan_states(U, psi0, out=st)
    torch.cuda.synchronize()
    print("ok", w.name, w.batch, w.K, w.L, float(np.abs(st[0, -1].cpu().numpy()).sum()))


if __name__ == "__main__":
    main()
