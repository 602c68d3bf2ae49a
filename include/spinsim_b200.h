/* spinsim_b200.h — C ABI of the B200-native Spinsim hot path (arXiv 2204.05586).
 *
 * Integrates the time-dependent Schrödinger equation i dψ/dt = H(t)ψ (Eq. schroedinger) for
 * spin-half (dim 2) and spin-one (dim 3) systems, H = ωx Jx + ωy Jy + ωz Jz + ωq Q, over a batch of
 * independent parameter sweeps:
 *   - one GPU thread owns one coarse interval [t_k, t_k + Δt] and runs L = Δt/δt fine steps
 *      of the commutator-free 4th-order Magnus method CF4 (Eq. cf4_implementation) inside a
 *     per-interval rotating frame;
 *   - exponentials are closed-form SU(2) for spin-half or Lie–Trotter with τ residual squarings for
 *     spin-one;
 *   - the interval unitaries U_k are chained into states ψ_{k+1} = U_k ψ_k (Eq. integration_compilation)
 *     by a decoupled-look-back matrix-product scan on the GPU.
 *
 * Conventions (every entry point):
 *   - Status: 0 = SS_OK, negative = error; ss_last_error() returns a thread-local message naming the offending
 *     argument.  Argument errors are detected synchronously before any launch; CUDA launch errors are reported as
 *     SS_ERR_CUDA by the call that detects them.  No entry point falls back to the CPU.
 *   - Memory: pointers prefixed d_ are CUDA device pointers, h_ are host pointers.  The caller owns every data
 *     buffer and the workspace; the library owns only the ss_sim handle (and, for ss_evaluate_host, device
 *     staging buffers cached inside it).  Device entry points never allocate.
 *   - Layout: row-major; complex numbers are interleaved (re, im) float64 pairs ("complex128"):
 *       sweep      [batch][P] float64, P = ss_num_sweep_params(field)
 *       state      [batch][dim] complex128
 *       states     [batch][K+1][dim] complex128, states[b][0] = state_init[b], states[b][k+1] = U_k states[b][k]
 *       unitaries  [batch][K][dim][dim] complex128 (lab frame)
 *     Basis order: spin-half (↑, ↓); spin-one m = +1, 0, −1 (reading R5).
 *   - Time grid (reading R7): K = (time_end − time_start)/Δt and L = Δt/δt must be integers within 1e-9
 *     relative (else SS_ERR_INVALID); Δt = time_step_output; δt = Δt / L; t_k = time_start + k·Δt.
 *   - Streams: `stream` is a cudaStream_t passed as void* (NULL = legacy default stream); all device work is
 *     stream-ordered and asynchronous unless stated.
 *   - Precision: `precision` selects only the fine-step arithmetic; all I/O is float64/complex128.
 */
#ifndef SPINSIM_B200_H
#define SPINSIM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  SS_OK = 0,
  SS_ERR_INVALID = -1,      /* bad argument (names it in ss_last_error) */
  SS_ERR_UNSUPPORTED = -2,  /* valid but unsupported combination */
  SS_ERR_CUDA = -3,         /* CUDA runtime / launch error, or no CUDA device */
  SS_ERR_NONFINITE = -4     /* non-finite sweep parameter or initial state */
};

enum ss_spin { SS_SPIN_HALF = 1, SS_SPIN_ONE = 2 };                 /* 2j */
enum ss_integration { SS_CF4 = 0, SS_MIDPOINT = 1, SS_HEUN = 2 };   /* P:323; Euler samplers P:702-704 */
/* SS_EXP_LIE_TROTTER_SU3: general spin-one Hamiltonians over the full su(3) basis (the paper
 * ships such an exponentiator without describing it — DESIGN.md readings R19, R20):
 *   H = ωx Jx + ωy Jy + ωz Jz + ωq Q + ωu1 U1 + ωu2 U2 + ωv1 V1 + ωv2 V2,
 *   U1 = Jx² − Jy², U2 = JxJy + JyJx (Δm = ±2), V1 = JxJz + JzJx, V2 = JyJz + JzJy (Δm = ±1);
 * Lie–Trotter U = T^n, n = 2^τ with the factor taken on the tridiagonalised generator: the
 * unitary similarity W (reading R20) makes S = W†HW real symmetric tridiagonal, T = W e^{−iD/2} e^{−iX}
 * e^{−iD/2} W† (D = diag S, X the (0,1)/(1,2) couplings of S, each ÷ n) — the shape of the paper's own factor
 * (Eq. lie_trotter_4) — then τ residual squarings of the complex-symmetric T₀ in double-angle form.  A second-order
 * splitting like the paper's basis product (which the oracle implements); the two agree to rounding for τ ≳ 20.
 * Spin-one only; accepts every field. */
enum ss_expo { SS_EXP_ANALYTIC = 0, SS_EXP_LIE_TROTTER = 1, SS_EXP_LIE_TROTTER_SU3 = 2 };  /* P:359 / P:360-466 / P:478 */
enum ss_precision { SS_FP64 = 0, SS_FP32 = 1 };
/* Built-in field functions replacing the paper's user numba function.  Sweep parameters:
 *   SS_FIELD_CONSTANT       [ωx, ωy, ωz, ωq]
 *   SS_FIELD_RABI_LINEAR    [ω0, Ω]            H = ω0 Jz + 2Ω cos(ω0 t) Jx
 *   SS_FIELD_RABI_CIRCULAR  [ω0, Ω]            H = ω0 Jz + Ω(cos(ω0 t) Jx + sin(ω0 t) Jy)
 *   SS_FIELD_NEURAL         [ω_bias, ω_rf, Ω, Ω_p, ω_sig, t_p, ω_q]
 *        H = ω_bias Jz + 2Ω cos(ω_rf t) Jx + Ω_p sinp(ω_sig (t − t_p)) Jz + ω_q Q   (Eq. neural_pulse)
 *   SS_FIELD_GRADIENT       [x, y]             ω_z = x − 2y
 * General spin-one fields (only with SS_EXP_LIE_TROTTER_SU3):
 *   SS_FIELD_SU3_CONSTANT   [ωx, ωy, ωz, ωq, ωu1, ωu2, ωv1, ωv2]
 *   SS_FIELD_SU3_DRIVE      [ω0, ω_q, Ω_x, Ω_v, Ω_u, ω_d]
 *        H = ω0 Jz + ω_q Q + Ω_x(cos ω_d t Jx + sin ω_d t Jy) + Ω_v(cos ω_d t V1 + sin ω_d t V2)
 *            + Ω_u(cos 2ω_d t U1 + sin 2ω_d t U2)     (upper/lower-pair couplings Ω_x ± Ω_v, two-photon Ω_u) */
enum ss_field {
  SS_FIELD_CONSTANT = 0,
  SS_FIELD_RABI_LINEAR = 1,
  SS_FIELD_RABI_CIRCULAR = 2,
  SS_FIELD_NEURAL = 3,
  SS_FIELD_GRADIENT = 4,
  SS_FIELD_USER = 5,        /* set by ss_create_user; not accepted by ss_create */
  SS_FIELD_SU3_CONSTANT = 6,
  SS_FIELD_SU3_DRIVE = 7
};

/* Simulator description (mirrors spinsim.Simulator's constructor arguments). */
typedef struct {
  int32_t spin;               /* ss_spin */
  int32_t integration;        /* ss_integration */
  int32_t exponentiation;     /* ss_expo; SPIN_HALF requires ANALYTIC; SPIN_ONE accepts both (ANALYTIC iff ω_q ≡ 0) */
  int32_t trotter_cutoff;     /* τ: n = 2^τ squarings' exponent; 0..60; default 24 */
  int32_t use_rotating_frame; /* 0/1; default 1 */
  int32_t precision;          /* ss_precision; SS_FP32 requires use_rotating_frame = 1 (else SS_ERR_UNSUPPORTED: in the
                                 lab frame FP32 rounding accumulates past its 1e-4 bar) */
  int32_t field;              /* ss_field */
} ss_sim_desc;

typedef struct ss_sim ss_sim;  /* opaque handle, owned by the library */

/* Create / destroy a simulator.  Validates the combination; no CUDA call is made. */
int ss_create(const ss_sim_desc* desc, ss_sim** out);
void ss_destroy(ss_sim* sim);

/* Create a simulator whose field function is user code compiled at run time (the paper's
 * user-supplied field functions).  `field_source` is CUDA C++ that defines
 *     __device__ void user_field(double t_k, double off, const double* p, double f[4])
 * writing f = (ωx, ωy, ωz, ωq) — with SS_EXP_LIE_TROTTER_SU3 f has 8 entries, + (ωu1, ωu2, ωv1, ωv2) — in rad/s at
 * time t_k + off (t_k = interval start, off = offset inside the interval,
 * kept apart so phases of fast drives can be formed accurately; f is zeroed before the call) for the sweep parameters
 * p[0 .. n_params), 1 ≤ n_params ≤ 64.  NVRTC compiles it with the library's own interval kernel for sm_100a (first call per simulator:
 * ~1 s); the rest of the description (spin, integration, exponentiation, τ, frame, precision) is honoured as for
 * built-in fields.  desc->field is ignored.  Compile errors return SS_ERR_INVALID with the NVRTC log in
 * ss_last_error().  Needs a CUDA device (SS_ERR_CUDA otherwise).  The analytic spin-one exponentiator is rejected
 * (ω_q ≡ 0 cannot be verified for user code). */
int ss_create_user(const ss_sim_desc* desc, const char* field_source, int32_t n_params, ss_sim** out);

/* Compile-only check of a user field (no device needed): SS_OK, or SS_ERR_INVALID with the NVRTC log in
 * ss_last_error(). */
int ss_compile_user_field(const ss_sim_desc* desc, const char* field_source, int32_t n_params);

/* Number of sweep parameters P of a built-in field (negative if unknown). */
int ss_num_sweep_params(int32_t field);

/* State dimension of a simulator: 2 (spin-half) or 3 (spin-one). */
int ss_dim(const ss_sim* sim);

/* Plan the time grid (reading R7): writes K, L and δt = Δt/L.  Pure host arithmetic. */
int ss_plan(double time_start, double time_end, double time_step_integration, double time_step_output,
            int64_t* K, int64_t* L, double* dt_fine);

/* Device workspace needed by ss_evaluate for `batch` sweeps of K intervals; includes room for the interval
 * unitaries when the caller passes d_unitaries = NULL, and — below the chain kernel's 4096 sweeps — for the fused
 * path's run aggregates and run start states (at most ⌈K/4⌉ + ⌈K/4⌉ + 1 per sweep). */
size_t ss_workspace_bytes(const ss_sim* sim, int64_t batch, int64_t K, int32_t unitaries_in_workspace);

/* Whole hot path on device buffers: interval kernel (§8(a) rows a1–a8) then the state scan (a9).
 *   d_sweep       device [batch][P] float64
 *   d_state_init  device [batch][dim] complex128
 *   d_states      device [batch][K+1][dim] complex128 (out)
 *   d_unitaries   device [batch][K][dim][dim] complex128 (out) or NULL (then kept in the workspace)
 *   d_workspace   device, >= ss_workspace_bytes(sim, batch, K, d_unitaries == NULL), 256-byte aligned
 * With d_unitaries == NULL on the SU(2)-form paths (spin-half; ANALYTIC spin-one) the interval operators reach the
 * scan in the workspace as SU(2) elements (a, b) of U = [[a, b], [−b*, a*]] (32 B per interval instead of 64 / 144 B;
 * D¹ of it for spin-one, reading R14) — the same operators, so the states agree with the dense path to
 * rounding.  Long problems below 4096 sweeps (≥ 16 waves of interval threads at 4 intervals per thread, K divisible
 * by the run length) take the fused path (DESIGN.md §5 item 16): each interval-kernel thread computes ipt ∈ {4, 8,
 * 16, 32} consecutive U_k and their run product, a coarse scan over the run products gives the run start states, and
 * a run chain writes the states — U_k bit for bit as on the unfused path, states equal to rounding (a different
 * product association; the scan's association is never part of the contract).  Validates sweep/state finiteness
 * (and ω_q ≡ 0 for ANALYTIC spin-one) with a tiny device check that synchronises the stream once, unless disabled by
 * ss_set_validation(sim, 0). */
int ss_evaluate(ss_sim* sim, double time_start, double time_end, double time_step_integration,
                double time_step_output, int64_t batch, const double* d_sweep, const double* d_state_init,
                double* d_states, double* d_unitaries, void* d_workspace, size_t workspace_bytes, void* stream);

/* Enable (1, default) / disable (0) the synchronous input validation inside ss_evaluate (disable it to capture
 * ss_evaluate in a CUDA graph). */
int ss_set_validation(ss_sim* sim, int32_t enabled);

/* Profiling hook: `event` (a cudaEvent_t passed as void*, owned by the caller; NULL to clear) is recorded by every
 * later ss_evaluate (and every chunk of ss_evaluate_host) on its stream between the interval kernel and the state
 * scan, so a caller can time the two phases of one call with its own events around it.  No other effect. */
int ss_set_split_event(ss_sim* sim, void* event);

/* Interval kernel only (rows a1–a8) for global interval indices k ∈ [k_begin, k_begin + k_count) of a grid of K
 * intervals: writes d_unitaries [batch][k_count][dim][dim].  The time grid uses the global k, so a time partition
 * reproduces the single-GPU operators bit for bit.  No validation kernel, no synchronisation. */
int ss_compute_unitaries(ss_sim* sim, double time_start, double time_end, double time_step_integration,
                         double time_step_output, int64_t k_begin, int64_t k_count, int64_t batch,
                         const double* d_sweep, double* d_unitaries, void* stream);

/* State scan only (row a9): states[b][0] = state_init[b], states[b][k+1] = U[b][k] states[b][k] for
 * k < k_count.  The kernel follows the problem's shape (DESIGN.md §5 "State propagation"): a per-sweep chain for
 * batch ≥ 4096 (dense spin-one operators: ≥ 2304), one cooperative wave for operators that fit in L2, a decoupled-look-back tile scan (dense) or the
 * two-pass run scan (compact operators of ss_scan_states_su2) otherwise — the association of the products, and so
 * the last-ulp rounding of the states, depends on that choice.  d_workspace >= ss_scan_workspace_bytes(dim, batch,
 * k_count) (includes, below 4096 sweeps, the two-pass scan's run products and run states: ≤ ⌈k_count/4⌉ of each per
 * sweep, plus its coarse scan's workspace). */
size_t ss_scan_workspace_bytes(int32_t dim, int64_t batch, int64_t k_count);
int ss_scan_states(int32_t dim, int64_t batch, int64_t k_count, const double* d_unitaries,
                   const double* d_state_init, double* d_states, void* d_workspace, size_t workspace_bytes,
                   void* stream);

/* Row a9 with the expected spin projection ⟨J⟩ = (ψ†Jxψ, ψ†Jyψ, ψ†Jzψ) (the paper's lazily computed
 * observable) fused into the state write-out.  d_spin: device [batch][k_count+1][3]
 * float64 (8-byte aligned).  d_states may be NULL to write only ⟨J⟩ (24 B instead of 16·dim B per interval); at least
 * one of the two must be non-NULL.  Workspace as ss_scan_states. */
int ss_scan_states_spin(int32_t dim, int64_t batch, int64_t k_count, const double* d_unitaries,
                        const double* d_state_init, double* d_states, double* d_spin, void* d_workspace,
                        size_t workspace_bytes, void* stream);

/* Row a9 over compact SU(2) operators (the form the SU(2)-form interval kernels accumulate, DESIGN.md §5 items
 * 10-11): d_ops device [batch][k_count][2] complex128 holds (a, b) of U_k = [[a, b], [−b*, a*]] (|a|² + |b|² = 1 is
 * assumed, not checked); dim = 2 applies U_k, dim = 3 its spin-1 representation
 * D¹(U) = [[a², √2ab, b²], [−√2ab*, |a|²−|b|², √2a*b], [b*², −√2a*b*, a*²]] (reading R14).  d_states and d_spin as in
 * ss_scan_states_spin (either may be NULL, not both); workspace >= ss_scan_workspace_bytes(dim, batch, k_count). */
int ss_scan_states_su2(int32_t dim, int64_t batch, int64_t k_count, const double* d_ops, const double* d_state_init,
                       double* d_states, double* d_spin, void* d_workspace, size_t workspace_bytes, void* stream);

/* Time-partition pieces (multi-GPU, one long simulation).  Aggregate of a partition:
 * d_aggregate[b] = U[b][k_count−1] ⋯ U[b][0]  ([batch][dim][dim] complex128).
 * d_workspace >= ss_aggregate_workspace_bytes(dim, batch, k_count). */
size_t ss_aggregate_workspace_bytes(int32_t dim, int64_t batch, int64_t k_count);
int ss_chain_aggregate(int32_t dim, int64_t batch, int64_t k_count, const double* d_unitaries, double* d_aggregate,
                       void* d_workspace, size_t workspace_bytes, void* stream);

/* Carry of partition `part`: d_carry[b] = A_{part−1} ⋯ A_0 state_init[b], from the all-gathered aggregates
 * d_aggregates [n_parts][batch][dim][dim] (applied to the state in this fixed order on every rank, so every rank
 * computes bit-identical carries).  part = 0 copies state_init. */
int ss_compose_carry(int32_t dim, int64_t batch, int32_t n_parts, int32_t part, const double* d_aggregates,
                     const double* d_state_init, double* d_carry, void* stream);

/* Building block for element-wise parity: exp(−i(ax Jx + ay Jy + az Jz + aq Q)) for d_args [n][4] float64 (for
 * SS_EXP_LIE_TROTTER_SU3: [n][8], + au1 U1 + au2 U2 + av1 V1 + av2 V2), with the simulator's spin / exponentiation /
 * τ / precision; writes d_out [n][dim][dim] complex128. */
/* Number of Hamiltonian coefficients per exponent argument / field sample: 8 for SS_EXP_LIE_TROTTER_SU3, else 4. */
int ss_num_coefficients(const ss_sim* sim);
int ss_exponentiate(const ss_sim* sim, int64_t n, const double* d_args, double* d_out, void* stream);

/* Advisory Magnus-convergence diagnostic ("∫‖H‖₂ < ξ ≈ 1.08686870"; never blocks execution): for every fine
 * step the two-point Gauss–Legendre estimate δt·(‖H(t₁)‖₂ + ‖H(t₂)‖₂)/2 of ∫‖H‖₂ over the step, on the CF4 sample
 * times and in the frame the simulator integrates in, with the exact spectral norm; d_out[b] (device, [batch]
 * float64) = the maximum over the steps of sweep b.  Convergence is indicated by d_out[b] < SS_MAGNUS_XI.  Works for
 * built-in and user (NVRTC) fields. */
#define SS_MAGNUS_XI 1.08686870
int ss_magnus_bound(ss_sim* sim, double time_start, double time_end, double time_step_integration,
                    double time_step_output, int64_t batch, const double* d_sweep, double* d_out, void* stream);

/* Expected spin projection ⟨J⟩ = (ψ†Jxψ, ψ†Jyψ, ψ†Jzψ) for d_states [n][dim] complex128;
 * writes d_out [n][3] float64. */
int ss_spin_projection(int32_t spin, int64_t n, const double* d_states, double* d_out, void* stream);

/* End-to-end call on HOST buffers: copies h_sweep/h_state_init to the device, runs the path and copies the states
 * (and unitaries if h_unitaries != NULL) back, pipelined over `n_chunks` chunks on an internal compute stream and
 * copy stream so device→host copies overlap compute (n_chunks ≤ 0: automatic — ≈ 40 time chunks where they apply,
 * else 4 batch chunks): batch chunks of geometrically shrinking size (B/2, B/4, …), or —
 * for n_chunks ≥ 6 and either batch ≥ 4096 or long sweeps (≥ 6 waves of interval work per chunk, e.g. one sweep of
 * 1e6 intervals) — time chunks of all sweeps continued from a running carry (bit-identical to ss_evaluate for
 * batch ≥ 4096; equal to rounding otherwise: the single-sweep scan restarts from the carry).  Batches of ≤ 4 sweeps
 * whose interval work spans ≥ 1.2 waves but is too short for time chunks (the paper's benchmark, one sweep of 1e5
 * intervals) take two wave-aligned time chunks instead — all whole waves but the last, then the rest — unless
 * n_chunks == 1 (one chunk, no pipelining).  Synchronous: returns after the results are in host memory.  Device
 * buffers are allocated once and cached in `sim`.  Pinned host buffers give full copy bandwidth. */
int ss_evaluate_host(ss_sim* sim, double time_start, double time_end, double time_step_integration,
                     double time_step_output, int64_t batch, const double* h_sweep, const double* h_state_init,
                     double* h_states, double* h_unitaries, int32_t n_chunks);

/* The chunk plan ss_evaluate_host uses for these arguments (pure host logic; needs no GPU — the SM count defaults to
 * 148 without one).  *kind: 0 = batch chunks (sizes[c] = sweeps), 1 = tent-shaped time chunks, 2 = the wave-aligned
 * time pair (sizes[c] = intervals of every sweep); *count = number of chunks.  sizes[0..cap) is caller-owned host
 * memory; SS_ERR_INVALID if cap < *count (then *count is still set) or on the time-grid errors of ss_plan. */
int ss_host_chunk_plan(const ss_sim* sim, double time_start, double time_end, double time_step_integration,
                       double time_step_output, int64_t batch, int32_t n_chunks, int32_t* kind, int64_t* sizes,
                       int32_t cap, int32_t* count);

/* Number of CUDA kernels this library has launched in the process so far (launch accounting for bench.py). */
int64_t ss_kernel_launches(void);

/* Thread-local description of the last error ("" if none). */
const char* ss_last_error(void);

/* ABI version (major*100 + minor). */
int ss_version(void);

#ifdef __cplusplus
}
#endif

#endif /* SPINSIM_B200_H */
