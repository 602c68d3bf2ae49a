"""CPU oracle for the Spinsim hot path (arXiv 2204.05586) — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may
import this module.  The product package ``paper_2204_05586_b200`` never imports it and shares no code with it.

This is a thin ctypes marshalling layer over ``liboracle.so`` (built from ``spinsim_oracle.cpp`` by ``build()``);
every computation happens in the C++ file, which cites the PAPER.md passage each step follows.

Parity status: every function here is pinned by ``tests/test_oracle_pins.py`` against closed forms, library
routines (scipy.linalg.expm), brute force or invariants fixed by the paper — see DESIGN.md §4.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "spinsim_oracle.cpp")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
# tests/test_oracle_mutations.py points this at a deliberately broken build to prove the pins catch it
_OVERRIDE = os.environ.get("SPINSIM_ORACLE_LIB")

SPIN = {"half": 1, "one": 2}
METHOD = {"cf4": 0, "midpoint": 1, "heun": 2}
EXPO = {"analytic": 0, "lie_trotter": 1, "lie_trotter_su3": 2}
FIELD = {"constant": 0, "rabi_linear": 1, "rabi_circular": 2, "neural": 3, "gradient": 4,
         "su3_constant": 6, "su3_drive": 7}
SU3_FIELDS = ("su3_constant", "su3_drive")     # fields with U1, U2, V1, V2 components (8 coefficients)

_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with g++ (plain C++17, -ffp-contract=off)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        cmd = ["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fPIC", "-shared", "-pthread",
               _SRC, "-o", _LIB_PATH]
        subprocess.check_call(cmd)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if _OVERRIDE:
        lib = ctypes.CDLL(_OVERRIDE)
    else:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
    d = ctypes.c_double
    i = ctypes.c_int
    ll = ctypes.c_longlong
    P = ctypes.c_void_p
    lib.oracle_constants.argtypes = [P]
    lib.oracle_num_params.argtypes = [i]
    lib.oracle_plan.argtypes = [d, d, d, d, ctypes.POINTER(ll), ctypes.POINTER(ll), ctypes.POINTER(d)]
    lib.oracle_grid.argtypes = [d, d, d, ll, ll, P]
    lib.oracle_field_sample.argtypes = [i, P, d, d, i, P]
    lib.oracle_rotating_frame.argtypes = [P, d, d, P]
    lib.oracle_exponentiate.argtypes = [i, i, i, i, ll, i, P, P]
    lib.oracle_trotter_residual_su3.argtypes = [P, i, P]
    lib.oracle_trotter_residual.argtypes = [d, d, d, d, P]
    lib.oracle_expm_dense.argtypes = [i, P, d, P]
    lib.oracle_fine_step.argtypes = [i, i, i, i, i, i, i, d, d, d, P, ll, ll, d, P]
    lib.oracle_evaluate.argtypes = [i, i, i, i, i, i, i, d, d, d, d, ll, P, P, P, P, i, ll, ll]
    lib.oracle_chain.argtypes = [i, ll, ll, P, P, P, P]
    lib.oracle_spin_projection.argtypes = [i, ll, P, P]
    lib.oracle_rms_error.argtypes = [ll, i, P, P]
    lib.oracle_magnus_bound.argtypes = [i, i, i, d, d, d, d, ll, P, P]
    lib.oracle_spectral_norm.argtypes = [i, P, P]
    lib.oracle_rms_error.restype = d
    _lib = lib
    return lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _c128(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.complex128))


def dim_of(spin: str) -> int:
    return 2 if spin == "half" else 3


def constants() -> dict:
    out = np.zeros(4)
    _load().oracle_constants(_ptr(out))
    return {"g1": out[0], "g2": out[1], "w_plus": out[2], "w_minus": out[3]}


def num_params(field: str) -> int:
    return _load().oracle_num_params(FIELD[field])


def plan(t0, t1, dt_int, dt_out):
    K, L, dt = ctypes.c_longlong(), ctypes.c_longlong(), ctypes.c_double()
    rc = _load().oracle_plan(t0, t1, dt_int, dt_out, ctypes.byref(K), ctypes.byref(L), ctypes.byref(dt))
    if rc != 0:
        raise ValueError("invalid time grid")
    return K.value, L.value, dt.value


def grid(t0, dt_out, dt_int, k, l):
    out = np.zeros(4)
    _load().oracle_grid(t0, dt_out, dt_int, k, l, _ptr(out))
    return {"t_k": out[0], "off1": out[1], "off2": out[2], "off_mid": out[3]}


def field_sample(field: str, params, t_k: float, off: float, long_double: bool = True) -> np.ndarray:
    """(ωx, ωy, ωz, ωq) — plus (ωu1, ωu2, ωv1, ωv2) for the su(3) fields — at t_k + off."""
    p = _f64(params)
    out = np.zeros(8)
    rc = _load().oracle_field_sample(FIELD[field], _ptr(p), t_k, off, int(long_double), _ptr(out))
    if rc != 0:
        raise ValueError(field)
    return out if field in SU3_FIELDS else out[:4]


def rotating_frame(f, t_local: float, omega_r: float) -> np.ndarray:
    """Field coefficients in the rotating frame; f has 4 or 8 entries (returned with the same length)."""
    f = _f64(f)
    n = f.shape[0]
    f8 = np.zeros(8)
    f8[:n] = f
    out = np.zeros(8)
    _load().oracle_rotating_frame(_ptr(f8), t_local, omega_r, _ptr(out))
    return out[:n]


def exponentiate(spin: str, args, expo: str = "analytic", tau: int = 24, long_double: bool = True) -> np.ndarray:
    """exp(−i(ax Jx + ay Jy + az Jz + aq Q [+ au1 U1 + au2 U2 + av1 V1 + av2 V2])) for args [n][4] (or [n][8] for
    the su(3) exponentiator); returns [n][dim][dim] complex128."""
    a = _f64(args)
    na = 8 if (a.ndim >= 1 and a.shape[-1] == 8) else 4
    a = np.ascontiguousarray(a.reshape(-1, na))
    d = dim_of(spin)
    out = np.zeros((a.shape[0], d, d), dtype=np.complex128)
    rc = _load().oracle_exponentiate(SPIN[spin], EXPO[expo], tau, int(long_double), a.shape[0], na, _ptr(a),
                                     _ptr(out))
    if rc != 0:
        raise ValueError("invalid exponentiator configuration")
    return out


def trotter_residual_su3(args, tau: int) -> np.ndarray:
    """T − I of the general spin-one factor — the paper's basis product in leapfrog order — for args [8]
    divided by n = 2^tau (reading R20)."""
    a = _f64(args).reshape(8)
    out = np.zeros((3, 3), dtype=np.complex128)
    _load().oracle_trotter_residual_su3(_ptr(a), tau, _ptr(out))
    return out


def trotter_residual(Phi, phi, z, q) -> np.ndarray:
    out = np.zeros((3, 3), dtype=np.complex128)
    _load().oracle_trotter_residual(Phi, phi, z, q, _ptr(out))
    return out


def expm_dense(H, s: float = 1.0) -> np.ndarray:
    """exp(−i s H) by long-double Taylor scaling and squaring (pins only)."""
    H = _c128(H)
    out = np.zeros_like(H)
    _load().oracle_expm_dense(H.shape[0], _ptr(H), s, _ptr(out))
    return out


def fine_step(spin, method, expo, tau, frame, field, params, t0, dt_out, dt_int, k, l, omega_r,
              long_double=True) -> np.ndarray:
    d = dim_of(spin)
    p = _f64(params)
    out = np.zeros((d, d), dtype=np.complex128)
    rc = _load().oracle_fine_step(SPIN[spin], METHOD[method], EXPO[expo], tau, int(frame), FIELD[field],
                                  int(long_double), t0, dt_out, dt_int, _ptr(p), k, l, omega_r, _ptr(out))
    if rc != 0:
        raise ValueError("invalid configuration")
    return out


def evaluate(spin="half", method="cf4", expo="analytic", tau=24, frame=True, field="neural", *, sweep,
             t0, t1, dt_int, dt_out, psi0, long_double=True, want_unitaries=True, nthreads=0,
             k_begin=0, k_end=-1):
    """Oracle evaluation.  sweep: [B][P]; psi0: [B][dim] complex.  Returns (states [B][nk+1][dim],
    unitaries [B][nk][dim][dim] or None) for intervals k in [k_begin, k_end)."""
    d = dim_of(spin)
    K, _, _ = plan(t0, t1, dt_int, dt_out)
    if k_end < 0:
        k_end = K
    nk = k_end - k_begin
    sw = _f64(sweep).reshape(-1, num_params(field))
    B = sw.shape[0]
    p0 = _c128(psi0).reshape(B, d)
    states = np.zeros((B, nk + 1, d), dtype=np.complex128)
    U = np.zeros((B, nk, d, d), dtype=np.complex128) if want_unitaries else None
    rc = _load().oracle_evaluate(SPIN[spin], METHOD[method], EXPO[expo], tau, int(frame), FIELD[field],
                                 int(long_double), t0, t1, dt_int, dt_out, B, _ptr(sw), _ptr(p0),
                                 _ptr(states), _ptr(U) if U is not None else None, nthreads, k_begin, k_end)
    if rc != 0:
        raise ValueError("oracle_evaluate rejected its arguments")
    return states, U


def chain(U, psi0, want_aggregate=False):
    """Sequential long-double chain ψ_{k+1} = U_k ψ_k.  U [B][K][d][d], psi0 [B][d]."""
    U = _c128(U)
    B, K, d, _ = U.shape
    p0 = _c128(psi0).reshape(B, d)
    states = np.zeros((B, K + 1, d), np.complex128)
    agg = np.zeros((B, d, d), np.complex128) if want_aggregate else None
    _load().oracle_chain(d, B, K, _ptr(U), _ptr(p0), _ptr(states), _ptr(agg) if agg is not None else None)
    return (states, agg) if want_aggregate else states


def spin_projection(spin: str, states) -> np.ndarray:
    d = dim_of(spin)
    s = _c128(states).reshape(-1, d)
    out = np.zeros((s.shape[0], 3))
    _load().oracle_spin_projection(SPIN[spin], s.shape[0], _ptr(s), _ptr(out))
    return out.reshape(np.asarray(states).shape[:-1] + (3,))


def rms_error(a, b) -> float:
    a = _c128(a)
    b = _c128(b)
    assert a.shape == b.shape
    return _load().oracle_rms_error(a.shape[0], a.shape[1], _ptr(a), _ptr(b))


MAGNUS_XI = 1.08686870


def magnus_bound(spin, frame, field, *, sweep, t0, t1, dt_int, dt_out) -> np.ndarray:
    """Per sweep: max over fine steps of δt·(‖H(t₁)‖₂ + ‖H(t₂)‖₂)/2 in the integration frame (P:304 diagnostic)."""
    sw = _f64(sweep).reshape(-1, num_params(field))
    out = np.zeros(sw.shape[0])
    rc = _load().oracle_magnus_bound(SPIN[spin], int(frame), FIELD[field], t0, t1, dt_int, dt_out, sw.shape[0],
                                     _ptr(sw), _ptr(out))
    if rc != 0:
        raise ValueError("oracle_magnus_bound rejected its arguments")
    return out


def spectral_norm(spin, f) -> float:
    """‖Σ f_j A_j‖₂ for 8 coefficients (spin-half uses the first three)."""
    f8 = np.zeros(8)
    f8[: len(f)] = f
    out = np.zeros(1)
    _load().oracle_spectral_norm(SPIN[spin], _ptr(f8), _ptr(out))
    return float(out[0])
