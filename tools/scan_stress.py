"""Scan-stress variant of C4: one spin-half sweep, 1 s at δt = 1 ns with Δt = 10 ns → K = 1e8
intervals, L = 10.  Times, with CUDA events:
  (a) the public two-call path — interval kernel writing dense U_k (64 B), then the single-sweep scan (scan3) over
      them: 96 B per interval (read U_k 64 B + write ψ 32 B);
  (b) ss_evaluate without U — the interval kernel hands the state pass compact SU(2) elements (32 B) and, fused, the
      run aggregates of its warps: 64 B per interval (read U 32 B + write ψ 32 B); (c) the same unfused; (d) dense U_k
      requested as an output (96 B per interval), fused.

    python tools/scan_stress.py > profiles/r02/<tag>/scan_stress.txt
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_05586_b200 as ss  # noqa: E402
import workloads as W  # noqa: E402

HBM = 6534.8e9


def main():
    w = W.c4_long(dt_int=1e-9, dt_out=10e-9, duration=1.0)
    sim = ss.Simulator(w.spin, w.method, w.expo, w.tau, w.frame, "fp64", w.field)
    sweep = torch.from_numpy(w.sweep).cuda()
    psi0 = torch.from_numpy(w.psi0).cuda()
    st = torch.empty((1, w.K + 1, 2), dtype=torch.complex128, device="cuda")
    print(f"C4 scan-stress: K = {w.K:.0e} intervals, L = {w.L}, {w.fine_steps:.0e} fine steps (spin-half, one sweep)")
    # (a) dense two-call path
    U = torch.empty((1, w.K, 2, 2), dtype=torch.complex128, device="cuda")
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
    print(f"(a) dense U:   interval kernel {t_int:.2f} ms ({w.fine_steps / (t_int * 1e-3):.3e} fine steps/s); scan "
          f"{t_scan:.3f} ms for {nbytes / 1e9:.1f} GB = {nbytes / (t_scan * 1e-3) / 1e9:.0f} GB/s "
          f"({nbytes / (t_scan * 1e-3) / HBM:.2f} of 6534.8 GB/s); step {t_int + t_scan:.2f} ms")
    del U, ws
    # (b)–(d) ss_evaluate: compact operators with the fused run aggregates (default), compact unfused
    # (SPINSIM_FUSED=0), dense U_k as an output with the fused path; the split between the interval kernel and the
    # state pass comes from the ss_set_split_event hook
    wsb = torch.empty(sim.workspace_bytes(1, w.K, True), dtype=torch.uint8, device="cuda")
    Ud = torch.empty((1, w.K, 2, 2), dtype=torch.complex128, device="cuda")
    sim.evaluate(sweep, w.t0, w.t0 + w.dt_out, w.dt_int, w.dt_out, psi0, want_unitaries=False)
    sim.set_validation(False)
    for tag, fused, dense in (("(b) compact, fused", "1", False), ("(c) compact, unfused", "0", False),
                              ("(d) dense U out, fused", "1", True)):
        os.environ["SPINSIM_FUSED"] = fused
        for rep in range(3):
            ev[0].record()
            sim.set_split_event(ev[1])
            sim.evaluate(sweep, w.t0, w.t1, w.dt_int, w.dt_out, psi0, want_unitaries=dense, workspace=wsb,
                         out_states=st, out_unitaries=Ud if dense else None)
            ev[2].record()
            torch.cuda.synchronize()
        sim.set_split_event(None)
        t_int, t_scan = ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])
        nbytes = w.K * (96 if dense else 64)
        print(f"{tag}: interval kernel {t_int:.2f} ms; states {t_scan:.3f} ms for {nbytes / 1e9:.1f} GB = "
              f"{nbytes / (t_scan * 1e-3) / 1e9:.0f} GB/s ({nbytes / (t_scan * 1e-3) / HBM:.2f} of 6534.8 GB/s); "
              f"step {t_int + t_scan:.2f} ms = {w.fine_steps / ((t_int + t_scan) * 1e-3):.3e} fine steps/s")
    os.environ.pop("SPINSIM_FUSED", None)
    print(f"final state norm − 1: {abs(torch.linalg.vector_norm(st[0, -1]).item() - 1):.2e}")


if __name__ == "__main__":
    main()
