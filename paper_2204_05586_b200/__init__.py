"""B200-native Spinsim hot path (arXiv 2204.05586): Python face of libspinsim_b200.so.

Thin wrappers over the C ABI in include/spinsim_b200.h (see _lib.py): they validate tensor shapes/dtypes/devices,
allocate outputs and workspace with torch on the current CUDA device and stream, and call the library.  Every step
of the method runs in the library's CUDA kernels; torch provides device memory, streams and process groups only.

    sim = Simulator(spin="one", exponentiation="lie_trotter", field="neural")
    res = sim.evaluate(sweep, 0.0, 0.1, 100e-9, 1e-6, state_init)     # sweep [B][P] f64, state_init [B][dim] c128 (cuda)
    res.state            # [B][K+1][dim] complex128 on the device
    res.time_evolution   # [B][K][dim][dim] complex128
    res.spin             # lazily computed ⟨J⟩ [B][K+1][3]

The argument names follow the paper's Simulator / evaluate / Results.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field as dc_field

import numpy as np
import torch

from . import _lib
from ._lib import EXPONENTIATION, FIELD, INTEGRATION, PRECISION, SPIN, SpinsimError, check

__all__ = ["Simulator", "Results", "SpinsimError", "plan", "num_sweep_params", "scan_states", "scan_states_spin",
           "scan_states_su2",
           "chain_aggregate",
           "compose_carry", "spin_projection", "kernel_launches", "load"]


def load():
    return _lib.load()


def _stream_ptr(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _dev_ptr(t: torch.Tensor, name: str, dtype=None, shape=None):
    """Device pointer of `t` after checking it: a contiguous CUDA tensor on the current device, of `dtype` and
    `shape` when given (raises before any library call, so the kernels never see a short or foreign buffer)."""
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor (there is no CPU path)")
    if t.device.index != torch.cuda.current_device():
        raise ValueError(f"{name} is on {t.device}, but the current CUDA device is cuda:{torch.cuda.current_device()}")
    if dtype is not None and t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _host_ptr(a: np.ndarray, name: str, dtype, shape):
    """Pointer of a host array after checking dtype, shape and C-contiguity (ss_evaluate_host reads/writes it raw)."""
    if not isinstance(a, np.ndarray) or a.dtype != dtype or tuple(a.shape) != tuple(shape) or not a.flags.c_contiguous:
        raise ValueError(f"{name} must be a C-contiguous {np.dtype(dtype)} array of shape {tuple(shape)}")
    if not a.flags.writeable and name.startswith("out"):
        raise ValueError(f"{name} must be writeable")
    return ctypes.c_void_p(a.ctypes.data)


def kernel_launches() -> int:
    """Number of CUDA kernels libspinsim_b200 has launched in this process."""
    return int(_lib.load().ss_kernel_launches())


def num_sweep_params(field: str) -> int:
    return int(_lib.load().ss_num_sweep_params(FIELD[field]))


def plan(time_start, time_end, time_step_integration, time_step_output):
    """(K, L, δt) of the time grid (reading R7); raises on a non-integral grid."""
    K, L, dt = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_double()
    check(_lib.load().ss_plan(time_start, time_end, time_step_integration, time_step_output, ctypes.byref(K),
                              ctypes.byref(L), ctypes.byref(dt)), "ss_plan")
    return K.value, L.value, dt.value


@dataclass
class Results:
    """Mirror of spinsim.Results: time, state, time-evolution operator and lazy spin projection."""
    time_start: float
    time_step_output: float
    spin_quantum: str
    state: torch.Tensor                      # [B][K+1][dim] complex128
    time_evolution: torch.Tensor | None      # [B][K][dim][dim] complex128
    _spin: torch.Tensor | None = dc_field(default=None, repr=False)

    @property
    def time(self) -> np.ndarray:
        K = self.state.shape[1] - 1
        return self.time_start + np.arange(K + 1) * self.time_step_output

    @property
    def spin(self) -> torch.Tensor:
        if self._spin is None:
            self._spin = spin_projection(self.spin_quantum, self.state)
        return self._spin


class Simulator:
    """Compiled-once simulator (the paper's spinsim.Simulator).  Kernels are specialised at build time
    for every (spin, exponentiator, integration method, field, precision); construction only picks them."""

    def __init__(self, spin="one", integration="cf4", exponentiation=None, trotter_cutoff=24,
                 use_rotating_frame=True, precision="fp64", field="neural", field_source=None, n_params=None):
        """field="user": `field_source` is CUDA C++ defining
        ``__device__ void user_field(double t_k, double off, const double* p, double f[4])`` (compiled at run time
        by NVRTC into the library's interval kernel; the paper's user field functions) and `n_params`
        the number of sweep parameters it reads.  exponentiation="lie_trotter_su3" (general spin-one)
        takes 8 Hamiltonian coefficients: the su3_* fields, or a user field writing f[8]."""
        if exponentiation is None:
            exponentiation = "analytic" if spin == "half" else "lie_trotter"
        self.spin, self.integration, self.exponentiation = spin, integration, exponentiation
        self.trotter_cutoff, self.use_rotating_frame = int(trotter_cutoff), bool(use_rotating_frame)
        self.precision, self.field = precision, field
        self.dim = 2 if spin == "half" else 3
        h = ctypes.c_void_p()
        lib = _lib.load()
        if field == "user":
            if field_source is None or n_params is None:
                raise ValueError('field="user" needs field_source and n_params')
            self.n_params = int(n_params)
            desc = _lib.ss_sim_desc(SPIN[spin], INTEGRATION[integration], EXPONENTIATION[exponentiation],
                                    int(trotter_cutoff), int(bool(use_rotating_frame)), PRECISION[precision], 0)
            check(lib.ss_create_user(ctypes.byref(desc), field_source.encode(), self.n_params, ctypes.byref(h)),
                  "ss_create_user")
        else:
            self.n_params = num_sweep_params(field)
            desc = _lib.ss_sim_desc(SPIN[spin], INTEGRATION[integration], EXPONENTIATION[exponentiation],
                                    int(trotter_cutoff), int(bool(use_rotating_frame)), PRECISION[precision],
                                    FIELD[field])
            check(lib.ss_create(ctypes.byref(desc), ctypes.byref(h)), "ss_create")
        self._h = h
        self._lib = lib

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._lib.ss_destroy(h)
            self._h = None

    def set_validation(self, enabled: bool) -> None:
        check(self._lib.ss_set_validation(self._h, int(bool(enabled))), "ss_set_validation")

    def set_split_event(self, event) -> None:
        """Profiling hook: record `event` (a torch.cuda.Event, or None to clear) inside every later evaluate() between
        the interval kernel and the state scan (ss_set_split_event)."""
        if event is not None and not event.cuda_event:
            event.record()                             # torch creates its CUDA events lazily, at the first record
        self._split_event = event                      # keep the torch event alive while the library holds it
        check(self._lib.ss_set_split_event(self._h, ctypes.c_void_p(event.cuda_event) if event is not None else None),
              "ss_set_split_event")

    def workspace_bytes(self, batch: int, K: int, unitaries_in_workspace: bool) -> int:
        return int(self._lib.ss_workspace_bytes(self._h, batch, K, int(unitaries_in_workspace)))

    def _check_sweep(self, sweep):
        if not isinstance(sweep, torch.Tensor) or sweep.dim() != 2 or sweep.shape[1] != self.n_params:
            raise ValueError(f"sweep must be [batch][{self.n_params}] float64 for field {self.field!r}")
        _dev_ptr(sweep, "sweep", torch.float64)
        return sweep.shape[0]

    def _check_inputs(self, sweep, state_init):
        B = self._check_sweep(sweep)
        _dev_ptr(state_init, "state_init", torch.complex128, (B, self.dim))
        return B

    def evaluate(self, sweep, time_start, time_end, time_step_integration, time_step_output, state_init,
                 want_unitaries=True, workspace=None, out_states=None, out_unitaries=None, stream=None) -> Results:
        """Whole hot path on device tensors (interval kernel + state scan)."""
        B = self._check_inputs(sweep, state_init)
        K, L, _ = plan(time_start, time_end, time_step_integration, time_step_output)
        dev = sweep.device
        states = out_states if out_states is not None else torch.empty((B, K + 1, self.dim), dtype=torch.complex128, device=dev)
        U = None
        if want_unitaries:
            U = out_unitaries if out_unitaries is not None else torch.empty((B, K, self.dim, self.dim), dtype=torch.complex128, device=dev)
        need = self.workspace_bytes(B, K, U is None)
        if workspace is None or workspace.numel() < need:
            workspace = torch.empty(need, dtype=torch.uint8, device=dev)
        check(self._lib.ss_evaluate(self._h, time_start, time_end, time_step_integration, time_step_output, B,
                                    _dev_ptr(sweep, "sweep"), _dev_ptr(state_init, "state_init"),
                                    _dev_ptr(states, "out_states", torch.complex128, (B, K + 1, self.dim)),
                                    _dev_ptr(U, "out_unitaries", torch.complex128, (B, K, self.dim, self.dim))
                                    if U is not None else None,
                                    _dev_ptr(workspace, "workspace", torch.uint8), workspace.numel(),
                                    _stream_ptr(stream)),
              "ss_evaluate")
        return Results(time_start, time_step_output, self.spin, states, U)

    def compute_unitaries(self, sweep, time_start, time_end, time_step_integration, time_step_output,
                          k_begin=0, k_count=None, out=None, stream=None) -> torch.Tensor:
        """Interval kernel only, for global intervals [k_begin, k_begin + k_count) → [B][k_count][dim][dim]."""
        B = self._check_sweep(sweep)
        K, _, _ = plan(time_start, time_end, time_step_integration, time_step_output)
        if k_count is None:
            k_count = K - k_begin
        U = out if out is not None else torch.empty((B, k_count, self.dim, self.dim), dtype=torch.complex128, device=sweep.device)
        check(self._lib.ss_compute_unitaries(self._h, time_start, time_end, time_step_integration, time_step_output,
                                             k_begin, k_count, B, _dev_ptr(sweep, "sweep"),
                                             _dev_ptr(U, "out", torch.complex128, (B, k_count, self.dim, self.dim)),
                                             _stream_ptr(stream)),
              "ss_compute_unitaries")
        return U

    @property
    def num_coefficients(self) -> int:
        """Hamiltonian coefficients per exponent argument: 8 for lie_trotter_su3, else 4."""
        return int(self._lib.ss_num_coefficients(self._h))

    def exponentiate(self, args: torch.Tensor, stream=None) -> torch.Tensor:
        """exp(−i(ax Jx + ay Jy + az Jz + aq Q [+ au1 U1 + au2 U2 + av1 V1 + av2 V2])) for args [n][4] (or [n][8] for
        lie_trotter_su3) float64 (device) → [n][dim][dim] complex128."""
        if not isinstance(args, torch.Tensor) or args.dim() != 2 or args.shape[1] != self.num_coefficients:
            raise ValueError(f"args must be [n][{self.num_coefficients}] for exponentiation {self.exponentiation!r}")
        args = args.contiguous()
        out = torch.empty((args.shape[0], self.dim, self.dim), dtype=torch.complex128, device=args.device)
        check(self._lib.ss_exponentiate(self._h, args.shape[0], _dev_ptr(args, "args", torch.float64),
                                        _dev_ptr(out, "out"), _stream_ptr(stream)), "ss_exponentiate")
        return out

    def magnus_bound(self, sweep: torch.Tensor, time_start, time_end, time_step_integration, time_step_output,
                     stream=None) -> torch.Tensor:
        """Advisory Magnus-convergence diagnostic: per sweep, the largest Gauss–Legendre estimate of ∫‖H‖₂
        over one fine step (in the integration frame); the expansion converges where it is < SS_MAGNUS_XI."""
        B = self._check_sweep(sweep)
        out = torch.empty(B, dtype=torch.float64, device=sweep.device)
        check(self._lib.ss_magnus_bound(self._h, time_start, time_end, time_step_integration, time_step_output, B,
                                        _dev_ptr(sweep, "sweep"), _dev_ptr(out, "out"), _stream_ptr(stream)),
              "ss_magnus_bound")
        return out

    def evaluate_host(self, sweep: np.ndarray, time_start, time_end, time_step_integration, time_step_output,
                      state_init: np.ndarray, out_states: np.ndarray | None = None, want_unitaries=False,
                      n_chunks: int = 0):
        """End-to-end call on host arrays (pinned for full bandwidth): H2D, kernels, D2H inside the library, pipelined
        over n_chunks chunks (0: automatic)."""
        K, _, _ = plan(time_start, time_end, time_step_integration, time_step_output)
        sweep = np.ascontiguousarray(sweep, dtype=np.float64)
        state_init = np.ascontiguousarray(state_init, dtype=np.complex128)
        if sweep.ndim != 2 or sweep.shape[1] != self.n_params:
            raise ValueError(f"sweep must be [batch][{self.n_params}] float64 for field {self.field!r}")
        B = sweep.shape[0]
        states = out_states if out_states is not None else np.empty((B, K + 1, self.dim), np.complex128)
        U = np.empty((B, K, self.dim, self.dim), np.complex128) if want_unitaries else None
        check(self._lib.ss_evaluate_host(self._h, time_start, time_end, time_step_integration, time_step_output, B,
                                         _host_ptr(sweep, "sweep", np.float64, (B, self.n_params)),
                                         _host_ptr(state_init, "state_init", np.complex128, (B, self.dim)),
                                         _host_ptr(states, "out_states", np.complex128, (B, K + 1, self.dim)),
                                         _host_ptr(U, "out_unitaries", np.complex128, (B, K, self.dim, self.dim))
                                         if U is not None else None, n_chunks), "ss_evaluate_host")
        return states, U

    def host_chunk_plan(self, time_start, time_end, time_step_integration, time_step_output, batch: int,
                        n_chunks: int = 0):
        """(kind, sizes) of the pipeline evaluate_host would run: kind "batch" (sizes in sweeps), "time" (tent) or
        "wave_pair" (sizes in intervals)."""
        kind, count = ctypes.c_int32(0), ctypes.c_int32(0)
        sizes = (ctypes.c_int64 * 64)()
        check(self._lib.ss_host_chunk_plan(self._h, time_start, time_end, time_step_integration, time_step_output,
                                           batch, n_chunks, ctypes.byref(kind), sizes, 64, ctypes.byref(count)),
              "ss_host_chunk_plan")
        return {0: "batch", 1: "time", 2: "wave_pair"}[kind.value], [int(x) for x in sizes[:count.value]]


def _unitaries_shape(unitaries):
    if not isinstance(unitaries, torch.Tensor) or unitaries.dim() != 4 or unitaries.shape[2] != unitaries.shape[3] \
            or unitaries.shape[2] not in (2, 3):
        raise ValueError("unitaries must be [batch][K][dim][dim] complex128, dim 2 or 3")
    B, K, dim, _ = unitaries.shape
    return B, K, dim


def scan_states(unitaries: torch.Tensor, state_init: torch.Tensor, out=None, workspace=None, stream=None) -> torch.Tensor:
    """ψ[b][0] = ψ0[b], ψ[b][k+1] = U[b][k] ψ[b][k] (decoupled look-back scan, row a9)."""
    B, K, dim = _unitaries_shape(unitaries)
    lib = _lib.load()
    need = int(lib.ss_scan_workspace_bytes(dim, B, K))
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(need, dtype=torch.uint8, device=unitaries.device)
    states = out if out is not None else torch.empty((B, K + 1, dim), dtype=torch.complex128, device=unitaries.device)
    check(lib.ss_scan_states(dim, B, K, _dev_ptr(unitaries, "unitaries", torch.complex128),
                             _dev_ptr(state_init, "state_init", torch.complex128, (B, dim)),
                             _dev_ptr(states, "out", torch.complex128, (B, K + 1, dim)),
                             _dev_ptr(workspace, "workspace", torch.uint8), workspace.numel(), _stream_ptr(stream)),
          "ss_scan_states")
    return states


def scan_states_spin(unitaries: torch.Tensor, state_init: torch.Tensor, want_states: bool = True, workspace=None,
                     stream=None):
    """Row a9 with ⟨J⟩ fused into the write-out: returns (states [B][K+1][dim] or None, spin [B][K+1][3])."""
    B, K, dim = _unitaries_shape(unitaries)
    lib = _lib.load()
    need = int(lib.ss_scan_workspace_bytes(dim, B, K))
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(need, dtype=torch.uint8, device=unitaries.device)
    states = torch.empty((B, K + 1, dim), dtype=torch.complex128, device=unitaries.device) if want_states else None
    spin = torch.empty((B, K + 1, 3), dtype=torch.float64, device=unitaries.device)
    check(lib.ss_scan_states_spin(dim, B, K, _dev_ptr(unitaries, "unitaries", torch.complex128),
                                  _dev_ptr(state_init, "state_init", torch.complex128, (B, dim)),
                                  _dev_ptr(states, "states") if states is not None else None, _dev_ptr(spin, "spin"),
                                  _dev_ptr(workspace, "workspace"), workspace.numel(), _stream_ptr(stream)),
          "ss_scan_states_spin")
    return states, spin


def scan_states_su2(ops: torch.Tensor, state_init: torch.Tensor, dim: int, want_states: bool = True,
                    want_spin: bool = False, workspace=None, stream=None):
    """Row a9 over compact SU(2) operators ops [B][K][2] complex128 = (a, b) of U = [[a, b], [−b*, a*]], applied
    directly (dim 2) or through D¹ (dim 3).  Returns (states [B][K+1][dim] or None, spin [B][K+1][3] or None)."""
    if not isinstance(ops, torch.Tensor) or ops.dim() != 3 or ops.shape[2] != 2 or dim not in (2, 3):
        raise ValueError("ops must be [batch][K][2] complex128 and dim 2 or 3")
    if not (want_states or want_spin):
        raise ValueError("want_states or want_spin must be set")
    B, K, _ = ops.shape
    lib = _lib.load()
    need = int(lib.ss_scan_workspace_bytes(dim, B, K))
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(need, dtype=torch.uint8, device=ops.device)
    states = torch.empty((B, K + 1, dim), dtype=torch.complex128, device=ops.device) if want_states else None
    spin = torch.empty((B, K + 1, 3), dtype=torch.float64, device=ops.device) if want_spin else None
    check(lib.ss_scan_states_su2(dim, B, K, _dev_ptr(ops, "ops", torch.complex128, (B, K, 2)),
                                 _dev_ptr(state_init, "state_init", torch.complex128, (B, dim)),
                                 _dev_ptr(states, "states") if states is not None else None,
                                 _dev_ptr(spin, "spin") if spin is not None else None,
                                 _dev_ptr(workspace, "workspace", torch.uint8), workspace.numel(), _stream_ptr(stream)),
          "ss_scan_states_su2")
    return states, spin


def chain_aggregate(unitaries: torch.Tensor, stream=None) -> torch.Tensor:
    """A[b] = U[b][K−1] ⋯ U[b][0] → [B][dim][dim]."""
    B, K, dim = _unitaries_shape(unitaries)
    lib = _lib.load()
    need = int(lib.ss_aggregate_workspace_bytes(dim, B, K))
    ws = torch.empty(need, dtype=torch.uint8, device=unitaries.device)
    out = torch.empty((B, dim, dim), dtype=torch.complex128, device=unitaries.device)
    check(lib.ss_chain_aggregate(dim, B, K, _dev_ptr(unitaries, "unitaries", torch.complex128), _dev_ptr(out, "out"),
                                 _dev_ptr(ws, "workspace"), need, _stream_ptr(stream)), "ss_chain_aggregate")
    return out


def compose_carry(aggregates: torch.Tensor, state_init: torch.Tensor, part: int, stream=None) -> torch.Tensor:
    """carry[b] = A_{part−1} ⋯ A_0 ψ0[b] from all-gathered aggregates [n_parts][B][dim][dim]."""
    if aggregates.dim() != 4 or aggregates.shape[2] != aggregates.shape[3] or aggregates.shape[2] not in (2, 3):
        raise ValueError("aggregates must be [n_parts][batch][dim][dim] complex128, dim 2 or 3")
    n_parts, B, dim, _ = aggregates.shape
    out = torch.empty((B, dim), dtype=torch.complex128, device=state_init.device)
    check(_lib.load().ss_compose_carry(dim, B, n_parts, part, _dev_ptr(aggregates, "aggregates", torch.complex128),
                                       _dev_ptr(state_init, "state_init", torch.complex128, (B, dim)),
                                       _dev_ptr(out, "carry"),
                                       _stream_ptr(stream)), "ss_compose_carry")
    return out


def spin_projection(spin: str, states: torch.Tensor, stream=None) -> torch.Tensor:
    """⟨J⟩ for states [..., dim] complex128 → [..., 3] float64."""
    states = states.contiguous()
    dim = states.shape[-1]
    if dim != (2 if spin == "half" else 3):
        raise ValueError(f"states of spin {spin!r} must end in dim {2 if spin == 'half' else 3}, got {dim}")
    n = states.numel() // dim
    out = torch.empty(states.shape[:-1] + (3,), dtype=torch.float64, device=states.device)
    check(_lib.load().ss_spin_projection(SPIN[spin], n, _dev_ptr(states, "states", torch.complex128),
                                         _dev_ptr(out, "out"), _stream_ptr(stream)), "ss_spin_projection")
    return out
