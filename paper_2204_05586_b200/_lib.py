"""ctypes binding of include/spinsim_b200.h — argument marshalling only.

Every function here has the name of the C entry point it wraps and does nothing but convert arguments (torch
tensors → device pointers, enums, the current CUDA stream) and turn a negative status into an exception carrying
ss_last_error().  All arithmetic of the method runs in libspinsim_b200.so's kernels.  There is no CPU fallback: if
the library is missing, loading raises; if no CUDA device is present, the library's entry points return
SS_ERR_CUDA and this binding raises.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# SPINSIM_LIB selects an in-tree tuning variant (build.py <variant> ...) for experiments; default is the product build.
LIB_PATH = os.environ.get("SPINSIM_LIB") or os.path.join(HERE, "libspinsim_b200.so")

SS_OK, SS_ERR_INVALID, SS_ERR_UNSUPPORTED, SS_ERR_CUDA, SS_ERR_NONFINITE = 0, -1, -2, -3, -4
SS_MAGNUS_XI = 1.08686870          # Magnus convergence radius
SPIN = {"half": 1, "one": 2}
INTEGRATION = {"cf4": 0, "midpoint": 1, "heun": 2}
EXPONENTIATION = {"analytic": 0, "lie_trotter": 1, "lie_trotter_su3": 2}
PRECISION = {"fp64": 0, "fp32": 1}
FIELD = {"constant": 0, "rabi_linear": 1, "rabi_circular": 2, "neural": 3, "gradient": 4, "su3_constant": 6,
         "su3_drive": 7}

# Every symbol include/spinsim_b200.h declares (tests/test_abi.py checks the header and the .so against this).
EXPORTS = [
    "ss_create", "ss_create_user", "ss_compile_user_field", "ss_destroy", "ss_num_sweep_params", "ss_dim", "ss_plan", "ss_workspace_bytes", "ss_evaluate",
    "ss_set_validation", "ss_compute_unitaries", "ss_scan_workspace_bytes", "ss_scan_states", "ss_scan_states_spin",
    "ss_aggregate_workspace_bytes", "ss_chain_aggregate", "ss_compose_carry", "ss_exponentiate",
    "ss_spin_projection", "ss_evaluate_host", "ss_kernel_launches", "ss_last_error", "ss_version",
    "ss_num_coefficients", "ss_magnus_bound", "ss_host_chunk_plan", "ss_set_split_event",
    "ss_scan_states_su2",
]


class SpinsimError(RuntimeError):
    def __init__(self, code: int, where: str, msg: str):
        super().__init__(f"{where} failed with status {code}: {msg}")
        self.code = code


class ss_sim_desc(ctypes.Structure):
    _fields_ = [("spin", ctypes.c_int32), ("integration", ctypes.c_int32), ("exponentiation", ctypes.c_int32),
                ("trotter_cutoff", ctypes.c_int32), ("use_rotating_frame", ctypes.c_int32),
                ("precision", ctypes.c_int32), ("field", ctypes.c_int32)]


_lib = None


def load() -> ctypes.CDLL:
    """Load libspinsim_b200.so (raises if it has not been built: run __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not found — build it with `python -m paper_2204_05586_b200.build`; "
                          "there is no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    i32, i64, d, P, sz = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p, ctypes.c_size_t
    sig = {
        "ss_create": (ctypes.c_int, [ctypes.POINTER(ss_sim_desc), ctypes.POINTER(P)]),
        "ss_create_user": (ctypes.c_int, [ctypes.POINTER(ss_sim_desc), ctypes.c_char_p, i32, ctypes.POINTER(P)]),
        "ss_compile_user_field": (ctypes.c_int, [ctypes.POINTER(ss_sim_desc), ctypes.c_char_p, i32]),
        "ss_destroy": (None, [P]),
        "ss_num_sweep_params": (ctypes.c_int, [i32]),
        "ss_dim": (ctypes.c_int, [P]),
        "ss_plan": (ctypes.c_int, [d, d, d, d, ctypes.POINTER(i64), ctypes.POINTER(i64), ctypes.POINTER(d)]),
        "ss_workspace_bytes": (sz, [P, i64, i64, i32]),
        "ss_evaluate": (ctypes.c_int, [P, d, d, d, d, i64, P, P, P, P, P, sz, P]),
        "ss_set_validation": (ctypes.c_int, [P, i32]),
        "ss_set_split_event": (ctypes.c_int, [P, P]),
        "ss_compute_unitaries": (ctypes.c_int, [P, d, d, d, d, i64, i64, i64, P, P, P]),
        "ss_scan_workspace_bytes": (sz, [i32, i64, i64]),
        "ss_scan_states": (ctypes.c_int, [i32, i64, i64, P, P, P, P, sz, P]),
        "ss_scan_states_spin": (ctypes.c_int, [i32, i64, i64, P, P, P, P, P, sz, P]),
        "ss_scan_states_su2": (ctypes.c_int, [i32, i64, i64, P, P, P, P, P, sz, P]),
        "ss_aggregate_workspace_bytes": (sz, [i32, i64, i64]),
        "ss_chain_aggregate": (ctypes.c_int, [i32, i64, i64, P, P, P, sz, P]),
        "ss_compose_carry": (ctypes.c_int, [i32, i64, i32, i32, P, P, P, P]),
        "ss_exponentiate": (ctypes.c_int, [P, i64, P, P, P]),
        "ss_spin_projection": (ctypes.c_int, [i32, i64, P, P, P]),
        "ss_evaluate_host": (ctypes.c_int, [P, d, d, d, d, i64, P, P, P, P, i32]),
        "ss_host_chunk_plan": (ctypes.c_int, [P, d, d, d, d, i64, i32, P, P, i32, P]),
        "ss_kernel_launches": (i64, []),
        "ss_last_error": (ctypes.c_char_p, []),
        "ss_version": (ctypes.c_int, []),
        "ss_num_coefficients": (ctypes.c_int, [P]),
        "ss_magnus_bound": (ctypes.c_int, [P, d, d, d, d, i64, P, P, P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def check(rc: int, where: str) -> None:
    if rc != SS_OK:
        raise SpinsimError(rc, where, load().ss_last_error().decode())
