"""Small end-to-end calls through every round-2 kernel path, for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): the fused interval kernel (compact and dense operators, both spins, every exponentiator, FP32), the coarse
scans, the warp-cooperative run chain (cp.async staging, in-place states), warp-shared trigonometry (full and partial
warps), the NVRTC user-field kernel in fused mode, and the chain kernel's per-sweep ring (several warps, ring wrap).

    compute-sanitizer --tool memcheck python tools/sanitize_paths.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_05586_b200 as ss  # noqa: E402
import workloads as W  # noqa: E402

USER = r"""
__device__ void user_field(double t_k, double off, const double* p, double f[4]) {
  f[0] = 2.0 * p[2] * cos(p[1] * (t_k + off)); f[2] = p[0]; f[3] = p[6];
}
"""


def run(w, precision="fp64", want_unitaries=False, field=None, **env):
    for k, v in env.items():
        os.environ[k] = str(v)
    if field == "user":
        sim = ss.Simulator(w.spin, w.method, w.expo, w.tau, w.frame, precision, "user", field_source=USER, n_params=7)
    else:
        sim = ss.Simulator(w.spin, w.method, w.expo, w.tau, w.frame, precision, w.field)
    res = sim.evaluate(torch.from_numpy(w.sweep).cuda(), w.t0, w.t1, w.dt_int, w.dt_out,
                       torch.from_numpy(w.psi0).cuda(), want_unitaries=want_unitaries)
    torch.cuda.synchronize()
    for k in env:
        del os.environ[k]
    return float(np.abs(res.state.cpu().numpy()).sum())


def main():
    half = W.c4_long(duration=256e-6, dt_int=200e-9).with_(
        sweep=np.repeat(W.c4_long().sweep, 3, 0), psi0=W.random_states(3, 2, 1))
    one_lt = W.c5_matrix("lie_trotter", batch=2).with_(t1=96e-6, dt_int=200e-9, psi0=W.random_states(2, 3, 2))
    one_an = W.c5_matrix("analytic", batch=3).with_(t1=160e-6, dt_int=200e-9, psi0=W.random_states(3, 3, 3))
    su3 = W.g1_su3(batch=2, duration=64e-6).with_(dt_int=200e-9, psi0=W.random_states(2, 3, 4))
    for w in (half, one_lt, one_an, su3):
        for wu in (False, True):
            for ipt in (4, 8, 32):
                run(w, want_unitaries=wu, SPINSIM_FUSED_IPT=ipt)
        run(w, SPINSIM_FUSED=0)
        for path in ("coop", "scan2", "scan3", "twopass", "chain"):
            run(w, SPINSIM_FUSED_IPT=8, SPINSIM_SCAN_PATH=path)
    run(one_lt, precision="fp32", SPINSIM_FUSED_IPT=8)
    run(one_an, precision="fp32", SPINSIM_FUSED_IPT=8)
    run(one_lt, field="user", SPINSIM_FUSED_IPT=8)
    # the standalone two-pass scan of compact operators (run products, coarse scan, run chain), K = 4·odd, 32·m
    for d in (2, 3):
        for B, K in ((3, 36 * 7), (2, 32 * 9)):
            q = np.random.default_rng(K).standard_normal((B, K, 4))
            q /= np.linalg.norm(q, axis=-1, keepdims=True)
            ops = np.stack([q[..., 0] + 1j * q[..., 1], q[..., 2] + 1j * q[..., 3]], -1)
            os.environ["SPINSIM_SCAN_PATH"] = "twopass"
            ss.scan_states_su2(torch.from_numpy(ops).cuda(), torch.from_numpy(W.random_states(B, d, 6)).cuda(), d,
                               want_spin=True)
            torch.cuda.synchronize()
            del os.environ["SPINSIM_SCAN_PATH"]
    # the chain kernel's per-sweep ring with several warps per CTA, a partial last CTA and the ring wrapping (dense
    # spin-one and spin-half operators, states and ⟨J⟩)
    for d in (2, 3):
        B, K = 601, 12 * 16 + 37
        z = np.random.default_rng(d).standard_normal((B, K, d, d, 2))
        U = np.linalg.qr(z[..., 0] + 1j * z[..., 1])[0]
        os.environ["SPINSIM_SCAN_PATH"] = "chain"
        ss.scan_states_spin(torch.from_numpy(U).cuda(), torch.from_numpy(W.random_states(B, d, 7)).cuda(),
                            want_states=True)
        torch.cuda.synchronize()
        del os.environ["SPINSIM_SCAN_PATH"]
    # a partial last warp (K·batch not a multiple of 32) and sweeps straddling warps: warp_trig's fallback
    run(W.c5_matrix("lie_trotter", batch=3).with_(t1=37e-6, psi0=W.random_states(3, 3, 5)))
    print("ok")


if __name__ == "__main__":
    main()
