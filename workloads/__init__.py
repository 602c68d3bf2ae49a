"""Seeded synthetic inputs for the Spinsim hot path — shared by tests, smoke() and bench.py.

This module holds NO arithmetic of the method (no field evaluation, no exponentials, no stepping): it only
builds input arrays — sweep-parameter tables, initial states, random exponent arguments — and names the
five BASELINE.json configurations C1–C5 (SURVEY.md §8(d) "Concrete synthetic inputs").  Both the oracle and
the CUDA path consume exactly these arrays.

Sweep-parameter layout per built-in field (same order on both sides):
  constant      [ωx, ωy, ωz, ωq]
  rabi_linear   [ω0, Ω]                         H = ω0 Jz + 2Ω cos(ω0 t) Jx
  rabi_circular [ω0, Ω]                         H = ω0 Jz + Ω(cos(ω0 t) Jx + sin(ω0 t) Jy)
  neural        [ω_bias, ω_rf, Ω, Ω_p, ω_sig, t_p, ω_q]
                H = ω_bias Jz + 2Ω cos(ω_rf t) Jx + Ω_p sinp(ω_sig (t − t_p)) Jz + ω_q Q   (Eq. neural_pulse)
  gradient      [x, y]                          ω_z = x − 2y
  su3_constant  [ωx, ωy, ωz, ωq, ωu1, ωu2, ωv1, ωv2]   general spin-one H, constant
  su3_drive     [ω0, ω_q, Ω_x, Ω_v, Ω_u, ω_d]   H = ω0 Jz + ω_q Q + Ω_x(cos ω_d t Jx + sin ω_d t Jy)
                + Ω_v(cos ω_d t V1 + sin ω_d t V2) + Ω_u(cos 2ω_d t U1 + sin 2ω_d t U2)   (reading R20)
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

TWO_PI = 2.0 * math.pi

# Eq. neural_pulse parameters: ω = 2π·700 kHz, Ω = 2π·1 kHz, Ω_p = 2π·70 Hz.
OMEGA_BIAS = TWO_PI * 700e3
OMEGA_DRESS = TWO_PI * 1e3
OMEGA_PULSE = TWO_PI * 70.0
# Quadratic shift for C2/C3 (reading R15: ⁸⁷Rb F=1, ≈72 Hz at the ≈1 G implied by 700 kHz).
OMEGA_Q = TWO_PI * 72.0

NUM_PARAMS = {"constant": 4, "rabi_linear": 2, "rabi_circular": 2, "neural": 7, "gradient": 2, "su3_constant": 8,
              "su3_drive": 6}


def neural_params(omega_bias=OMEGA_BIAS, omega_rf=None, omega_dress=OMEGA_DRESS, omega_pulse=OMEGA_PULSE,
                  omega_sig=OMEGA_DRESS, t_p=23.3e-3, omega_q=OMEGA_Q) -> np.ndarray:
    if omega_rf is None:
        omega_rf = omega_bias
    return np.array([omega_bias, omega_rf, omega_dress, omega_pulse, omega_sig, t_p, omega_q], dtype=np.float64)


@dataclasses.dataclass(frozen=True)
class Workload:
    name: str
    spin: str
    method: str
    expo: str
    tau: int
    frame: bool
    field: str
    t0: float
    t1: float
    dt_int: float
    dt_out: float
    sweep: np.ndarray          # [B][P] float64
    psi0: np.ndarray           # [B][dim] complex128

    @property
    def batch(self) -> int:
        return self.sweep.shape[0]

    @property
    def dim(self) -> int:
        return 2 if self.spin == "half" else 3

    @property
    def K(self) -> int:
        return int(round((self.t1 - self.t0) / self.dt_out))

    @property
    def L(self) -> int:
        return int(round(self.dt_out / self.dt_int))

    @property
    def fine_steps(self) -> int:
        return self.batch * self.K * self.L

    def with_(self, **kw) -> "Workload":
        return dataclasses.replace(self, **kw)

    def describe(self) -> dict:
        return {"workload": self.name, "spin": self.spin, "method": self.method, "exponentiator": self.expo,
                "trotter_cutoff": self.tau, "rotating_frame": self.frame, "field": self.field,
                "time_start": self.t0, "time_end": self.t1, "time_step_integration": self.dt_int,
                "time_step_output": self.dt_out, "batch": self.batch, "K": self.K, "L": self.L}


def basis_state(dim: int, batch: int = 1) -> np.ndarray:
    psi = np.zeros((batch, dim), dtype=np.complex128)
    psi[:, 0] = 1.0
    return psi


def random_states(batch: int, dim: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    z = rng.standard_normal((batch, dim)) + 1j * rng.standard_normal((batch, dim))
    return z / np.linalg.norm(z, axis=1, keepdims=True)


def random_exponent_args(n: int, scale: float, seed: int, quad: bool = True) -> np.ndarray:
    """(ax, ay, az, aq) uniform in [−scale, scale]^4 (the paper's random-matrix exponentiator test)."""
    rng = np.random.default_rng(seed)
    a = rng.uniform(-scale, scale, size=(n, 4))
    if not quad:
        a[:, 3] = 0.0
    return a


def random_exponent_args_su3(n: int, scale: float, seed: int) -> np.ndarray:
    """All 8 su(3) coefficients (ax, ay, az, aq, au1, au2, av1, av2) uniform in [−scale, scale]^8."""
    rng = np.random.default_rng(seed)
    return rng.uniform(-scale, scale, size=(n, 8))


def su3_drive_params(omega0=OMEGA_BIAS, omega_q=OMEGA_Q, omega_x=OMEGA_DRESS, omega_v=0.4 * OMEGA_DRESS,
                     omega_u=0.25 * OMEGA_DRESS, omega_d=None) -> np.ndarray:
    """[ω0, ω_q, Ω_x, Ω_v, Ω_u, ω_d]: unequal couplings of the upper/lower pairs (Ω_x ± Ω_v) plus a two-photon
    drive Ω_u; ω_d = ω0 (resonant) unless given."""
    if omega_d is None:
        omega_d = omega0
    return np.array([omega0, omega_q, omega_x, omega_v, omega_u, omega_d], dtype=np.float64)


# ---------------------------------------------------------------------------------------------------------
# BASELINE.json configs.
# ---------------------------------------------------------------------------------------------------------
def c1_rabi(field: str = "rabi_circular") -> Workload:
    """C1: spin-half Rabi flop, 1 ms, δt = 100 ns, Δt = 1 µs, single simulation."""
    return Workload("C1", "half", "cf4", "analytic", 24, True, field, 0.0, 1e-3, 100e-9, 1e-6,
                    np.array([[OMEGA_BIAS, OMEGA_DRESS]]), basis_state(2))


def c2_neural(dt_int: float = 100e-9, duration: float = 0.1) -> Workload:
    """C2: spin-one neural-sensing benchmark (Eq. neural_pulse + quadratic shift), 100 ms, Lie–Trotter τ=24."""
    return Workload("C2", "one", "cf4", "lie_trotter", 24, True, "neural", 0.0, duration, dt_int, 1e-6,
                    neural_params(t_p=23.3e-3)[None, :], basis_state(3))


def c3_sweep_params(n_dress: int = 64, n_detune: int = 128) -> np.ndarray:
    """8192 = 64 dressing amplitudes Ω ∈ linspace(0.5, 1.5)·2π kHz × 128 detunings Δ ∈ linspace(−2, 2)·2π kHz,
    row-major with Ω outer; ω_rf = ω_bias + Δ.  t_p = 2.33 ms for the 10 ms window (reading R11)."""
    dress = np.linspace(0.5, 1.5, n_dress) * TWO_PI * 1e3
    detune = np.linspace(-2.0, 2.0, n_detune) * TWO_PI * 1e3
    rows = []
    for om in dress:
        for de in detune:
            rows.append(neural_params(omega_rf=OMEGA_BIAS + de, omega_dress=om, t_p=2.33e-3))
    return np.stack(rows)


def c3_batched(batch: int = 8192, duration: float = 0.01) -> Workload:
    """C3: batched parameter sweep, spin-one, 10 ms each, δt = 100 ns, Δt = 1 µs (K = 1e4, L = 10)."""
    sweep = c3_sweep_params()
    if batch <= sweep.shape[0]:
        sweep = sweep[:batch]
    else:                                   # weak-scaling blocks beyond 8192 repeat the grid
        sweep = np.concatenate([sweep] * int(math.ceil(batch / sweep.shape[0])))[:batch]
    return Workload("C3", "one", "cf4", "lie_trotter", 24, True, "neural", 0.0, duration, 100e-9, 1e-6,
                    np.ascontiguousarray(sweep), basis_state(3, sweep.shape[0]))


def c4_long(duration: float = 1.0, dt_int: float = 1e-9, dt_out: float = 1e-6) -> Workload:
    """C4: single long spin-half simulation, 1 s at δt = 1 ns (t_p = 233 ms as printed)."""
    return Workload("C4", "half", "cf4", "analytic", 24, True, "neural", 0.0, duration, dt_int, dt_out,
                    neural_params(t_p=0.233, omega_q=0.0)[None, :], basis_state(2))


def c5_matrix(expo: str = "lie_trotter", batch: int = 1) -> Workload:
    """C5: Eq. neural_pulse as printed (ω_q = 0, so the analytic spin-one exponentiator is valid), 100 ms,
    δt = 100 ns; throughput variant: 100 sweeps with Ω = linspace(0.9, 1.1, 100)·2π kHz."""
    if batch == 1:
        sweep = neural_params(t_p=23.3e-3, omega_q=0.0)[None, :]
    else:
        sweep = np.stack([neural_params(omega_dress=om, t_p=23.3e-3, omega_q=0.0)
                          for om in np.linspace(0.9, 1.1, batch) * TWO_PI * 1e3])
    return Workload("C5", "one", "cf4", expo, 24, True, "neural", 0.0, 0.1, 100e-9, 1e-6, sweep,
                    basis_state(3, batch))


def g1_su3(batch: int = 8192, duration: float = 0.01) -> Workload:
    """G1 (not a BASELINE config): a C3-shaped batched sweep of a general spin-one system —
    the su3_drive field (upper/lower-pair couplings Ω_x ± Ω_v, two-photon drive Ω_u, quadratic shift) through the
    su(3) Lie–Trotter exponentiator.  64 values Ω_v ∈ linspace(0, 0.8)·Ω_x × 128 drive detunings
    Δ ∈ linspace(−2, 2)·2π kHz (ω_d = ω0 + Δ), Ω_x = 2π·1 kHz, Ω_u = 2π·250 Hz; 10 ms, δt = 100 ns, Δt = 1 µs."""
    rows = []
    for ov in np.linspace(0.0, 0.8, 64) * OMEGA_DRESS:
        for de in np.linspace(-2.0, 2.0, 128) * TWO_PI * 1e3:
            rows.append(su3_drive_params(omega_v=ov, omega_d=OMEGA_BIAS + de))
    sweep = np.stack(rows)
    if batch <= sweep.shape[0]:
        sweep = sweep[:batch]
    else:
        sweep = np.concatenate([sweep] * int(math.ceil(batch / sweep.shape[0])))[:batch]
    return Workload("G1", "one", "cf4", "lie_trotter_su3", 24, True, "su3_drive", 0.0, duration, 100e-9, 1e-6,
                    np.ascontiguousarray(sweep), basis_state(3, sweep.shape[0]))


CONFIGS = {"C1": c1_rabi, "C2": c2_neural, "C3": c3_batched, "C4": c4_long, "C5": c5_matrix, "G1": g1_su3}
