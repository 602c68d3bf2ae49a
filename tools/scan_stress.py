"""Scan-stress variant of C4: one spin-half sweep, 1 s at δt = 1 ns with Δt = 10 ns → K = 1e8
intervals, L = 10.  Times the interval kernel and the single-sweep decoupled-look-back scan (scan3) separately and
reports the scan's HBM bandwidth (96 B per interval: read U_k 64 B + write ψ 32 B).

    python tools/scan_stress.py > profiles/r01/scan_stress.txt
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_05586_b200 as ss  # noqa: E402
import workloads as W  # noqa: E402


def main():
    w = W.c4_long(dt_int=1e-9, dt_out=10e-9, duration=1.0)
    sim = ss.Simulator(w.spin, w.method, w.expo, w.tau, w.frame, "fp64", w.field)
    sweep = torch.from_numpy(w.sweep).cuda()
    psi0 = torch.from_numpy(w.psi0).cuda()
    U = torch.empty((1, w.K, 2, 2), dtype=torch.complex128, device="cuda")
    st = torch.empty((1, w.K + 1, 2), dtype=torch.complex128, device="cuda")
    ws = torch.empty(int(ss._lib.load().ss_scan_workspace_bytes(2, 1, w.K)), dtype=torch.uint8, device="cuda")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    for rep in range(3):
        ev[0].record()
        sim.compute_unitaries(sweep, w.t0, w.t1, w.dt_int, w.dt_out, out=U)
        ev[1].record()
        ss.scan_states(U, psi0, out=st, workspace=ws)
        ev[2].record()
        torch.cuda.synchronize()
    t_int, t_scan = ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])
    nbytes = w.K * 96
    print(f"C4 scan-stress: K = {w.K:.0e} intervals, L = {w.L}, {w.fine_steps:.0e} fine steps (spin-half, one sweep)")
    print(f"interval kernel {t_int:.2f} ms ({w.fine_steps / (t_int * 1e-3):.3e} fine steps/s)")
    print(f"scan (single-sweep decoupled look-back) {t_scan:.2f} ms for {nbytes / 1e9:.1f} GB = "
          f"{nbytes / (t_scan * 1e-3) / 1e9:.0f} GB/s ({nbytes / (t_scan * 1e-3) / 6534.8e9:.2f} of 6534.8 GB/s)")
    print(f"final state norm − 1: {abs(torch.linalg.vector_norm(st[0, -1]).item() - 1):.2e}")


if __name__ == "__main__":
    main()
