"""Mutation check for the oracle pins: plausible transcription mistakes in oracle/spinsim_oracle.cpp (a dropped
term, a wrong sign, a transposed operand, a misprint left in) must each make tests/test_oracle_pins.py fail.
Each mutant is compiled to a temporary library and the pins are run against it in a subprocess."""
import os
import subprocess
import sys
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "spinsim_oracle.cpp")

MUTANTS = {
    # CF4 factor order swapped: exp(−iH̄1δt) exp(−iH̄2δt) (drops to 2nd order, SURVEY [V12])
    "cf4_order": ("return mul(e2, e1);", "return mul(e1, e2);"),
    # the misprinted T22 = cosΦ e^{i4q} of Eq. lie_trotter_4 left in
    "t22_misprint": ("a.a[1][1] = expm1i(th2) - R(2) * s * s * std::exp(I * th2);",
                     "a.a[1][1] = std::cos(Phi) * std::exp(I * R(4) * q) - R(1);"),
    # the misprinted T13 phase sign left in
    "t13_misprint": ("a.a[0][2] = -((s * eq6_m * em_phi) * (s * eq6_m * em_phi));",
                     "a.a[0][2] = -((s * eq6_p * em_phi) * (s * eq6_p * em_phi));"),
    # frame rotation direction flipped
    "frame_sign": ("f[0] = c * fx + s * fy;\n  f[1] = -s * fx + c * fy;", "f[0] = c * fx - s * fy;\n  f[1] = s * fx + c * fy;"),
    # frame exit forgotten sign: R(+Δt) instead of R(−Δt)
    "exit_sign": ("std::exp(-I * omega_r * m * (R)g.dt_out)", "std::exp(I * omega_r * m * (R)g.dt_out)"),
    # residual squaring (a + 2I)a with the 2I dropped
    "residual_drop_2I": ("b.a[i][i] += R(2);", "b.a[i][i] += R(1);"),
    # CF4 weights transposed: H̄1 gets w− on f1
    "weights_swapped": ("a1[j] = (wp * f1[j] + wm * f2[j]) * dt;", "a1[j] = (wm * f1[j] + wp * f2[j]) * dt;"),
    # accumulate u on the wrong side (postmultiply)
    "postmultiply": ("U = mul(u, U);", "U = mul(U, u);"),
    # ω_r sampled at the interval start instead of the midpoint
    "omega_r_start": ("field_sample<R>(c.field, p, t_k, 0.5 * g.dt_out, f);", "field_sample<R>(c.field, p, t_k, 0.0, f);"),
    # SU(2) closed form with cos(r) instead of cos(r/2)
    "su2_halfangle": ("const R c = std::cos(r / R(2));", "const R c = std::cos(r);"),
    # spin-one Jy sign convention broken inside the analytic map
    "d1_sign": ("D.a[1][0] = -rt2 * al * std::conj(be);", "D.a[1][0] = rt2 * al * std::conj(be);"),
    # --- general spin-one (su(3)) exponentiator and fields (readings R19, R20) ---
    # V1 built from the wrong pair of spin matrices (operator mix-up in the basis, reading R19)
    "su3_v1_def": ("b.A[6] = anti(Jx, Jz);", "b.A[6] = anti(Jy, Jz);"),
    # U2 = JxJy only: not Hermitian
    "su3_u2_herm": ("b.A[5] = anti(Jx, Jy);", "b.A[5] = mul(Jx, Jy);"),
    # U pair rotated by θ instead of 2θ in the frame
    "su3_u_frame_angle": ("const R c2 = std::cos(R(2) * th), s2 = std::sin(R(2) * th);", "const R c2 = c, s2 = s;"),
    # leapfrog half-step dropped on the outer factors of the first half (over-rotation)
    "su3_outer_half": ("for (int q = 0; q < 7; ++q) t = res_prod(t, factor(outer[q], R(0.5)));",
                       "for (int q = 0; q < 7; ++q) t = res_prod(t, factor(outer[q], R(1)));"),
    # middle factor multiplied on the wrong side: no longer symmetric (first-order splitting)
    "su3_middle_side": ("t = res_prod(t, factor(middle, R(1)));", "t = res_prod(factor(middle, R(1)), t);"),
    # closed form with cos θ − 1 = −sin²(θ/2) (dropped factor 2)
    "su3_cosm1": ("const R cosm1 = -R(2) * sh * sh, sn = std::sin(th);", "const R cosm1 = -sh * sh, sn = std::sin(th);"),
    # closed form with +i sin θ A
    "su3_sin_sign": ("e.a[i][j] = -I * sn * A.a[i][j] + cosm1 * A2.a[i][j];", "e.a[i][j] = I * sn * A.a[i][j] + cosm1 * A2.a[i][j];"),
    # two-photon drive at ω_d instead of 2ω_d
    "su3_drive_2w": ("f[4] = (R)p[4] * std::cos(R(2) * ph);", "f[4] = (R)p[4] * std::cos(ph);"),
    # --- Magnus diagnostic ---
    # coarse instead of fine step in the ∫‖H‖ estimate
    "magnus_dt": ("const R n = (R)g.dt_int * (spectral_norm", "const R n = (R)g.dt_out * (spectral_norm"),
    # wrong angle in the trigonometric cubic roots
    "spectral_root": ("const R phi = std::acos(c) / R(3),", "const R phi = std::acos(c) / R(2),"),
}


@pytest.mark.slow
@pytest.mark.parametrize("name", sorted(MUTANTS))
def test_pins_kill_mutant(name):
    old, new = MUTANTS[name]
    src = open(SRC).read()
    assert src.count(old) == 1, f"mutation anchor for {name} not found exactly once"
    with tempfile.TemporaryDirectory() as d:
        cpp = os.path.join(d, "m.cpp")
        so = os.path.join(d, "libm.so")
        open(cpp, "w").write(src.replace(old, new))
        subprocess.check_call(["g++", "-O1", "-std=c++17", "-ffp-contract=off", "-fPIC", "-shared", "-pthread",
                               cpp, "-o", so])
        env = dict(os.environ, SPINSIM_ORACLE_LIB=so)
        r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                            os.path.join(ROOT, "tests", "test_oracle_pins.py"),
                            os.path.join(ROOT, "tests", "test_oracle_pins_su3.py")],
                           env=env, cwd=ROOT, capture_output=True, text=True, timeout=600)
        assert r.returncode != 0, f"mutant {name} survived the pins:\n{r.stdout[-2000:]}"
