// interval_kernel.cuh — the per-interval unitary kernel (SURVEY §8(a) rows a1–a8).
//
// One thread ↔ one (sweep b, interval k): it enters the rotating frame at ω_r = ω_z(t_k + Δt/2)
// (P:539-541), runs the L fine steps of CF4 (Eq. cf4_implementation) — two Gauss-point field samples
// (P:325-329), frame rotation, weights, two exponentials, u = e₂e₁ premultiplied into U_r
// — holding U_r − I in registers in residual form (reading R9), and finally writes the lab-frame
// U_k = R_{ω_r}(−Δt) U_r (Eq. exit_rotating_frame).
//
// The work per thread is ~6e3 FP64 instructions per fine step for spin-one Lie–Trotter (93 % in the τ residual
// squarings), all register-resident: the kernel is FP64-pipe bound, so the launch is sized for
// occupancy with full ILP (18 independent accumulation chains per squaring) rather than for memory.
#pragma once

#include "ops.cuh"
#include "spinsim_device.cuh"

namespace ssb {

struct IntervalParams {
  double t0;          // time_start
  double dt_out;      // Δt
  double dt;          // δt = Δt/L
  double g1dt, g2dt;  // fl(g1·δt), fl(g2·δt)
  double half_dt;     // fl(0.5·δt)
  double half_dt_out; // fl(0.5·Δt)
  double wpd, wmd;    // fl(w±·δt): the CF4 weights with δt folded in (read from the parameter bank, no UMOV)
  int64_t L;
  int64_t k_begin, k_count, batch;
  int64_t n_threads;  // batch·k_stride: interval slots of the launch
  int64_t k_stride;   // thread slots per sweep: k_count, or ⌈k_count/ipt⌉ when run aggregates are written
  int64_t ipt;        // intervals per thread: 1, or the run length of the fused path (S = 1)
  int32_t tau;
  int32_t frame;
  int32_t split;        // S: lanes per interval (power of two ≤ 32); lane p runs fine steps [p·L/S, (p+1)·L/S)
  int32_t op_format;    // OP_DENSE, or OP_SU2 (SU(2)-form accumulators only): the layout of `unitaries`
  const double* sweep;  // [batch][P]
  double* unitaries;    // [batch][k_count][D][D] complex128 (OP_DENSE) or [batch][k_count][2] complex128 (OP_SU2)
  double* run_agg;      // NULL, or [batch][k_stride] operators (op_format): the product of each thread's ipt intervals
};

#ifndef SS_INTERVAL_THREADS
#define SS_INTERVAL_THREADS 128
#endif
constexpr int kIntervalThreads = SS_INTERVAL_THREADS;
// Resident blocks per SM requested from ptxas: 16 warps/SM (128 registers) without spills for every instance.
#ifndef SS_INTERVAL_MINBLOCKS
#define SS_INTERVAL_MINBLOCKS 4
#endif
// The general spin-one kernel holds a dense 3×3 residual (18 reals) plus the squaring's output copy beside the
// accumulator; SS_INTERVAL_MINBLOCKS_SU3 trades occupancy against spills for it (G1 on B200 with the closed-form
// factor: 2 → 2.63e9, 3 → 2.74e9, 4 → 2.70e9 fine steps/s; with the Taylor factor of §5 item 9: 3 → 3.08e9,
// 4 (128 registers, 316 B spilled) → 3.11e9).
#ifndef SS_INTERVAL_MINBLOCKS_SU3
#define SS_INTERVAL_MINBLOCKS_SU3 4
#endif
template <int SPIN, int EXPO, typename T> constexpr int kIntervalMinBlocks() {
  return EXPO == EXP_LIE_TROTTER_SU3 ? SS_INTERVAL_MINBLOCKS_SU3 : SS_INTERVAL_MINBLOCKS;
}

#ifndef SS_SU2_SHORT_BODIES
#define SS_SU2_SHORT_BODIES 1   // SU(2) short-series choice as specialised step bodies (1) or a run-time flag (0)
#endif
#ifndef SS_STEP_UNROLL
#define SS_STEP_UNROLL 1    // unroll of the rotated-phase steps between anchors (SU(2)-form paths; tuning knob)
#endif

template <int NC, int F>
__device__ __forceinline__ void sample_in_frame(const Field<F>& fld, double off, double omega_r, int frame,
                                                double* f) {
  fld.sample(off, f);
  if (frame) to_rotating_frame<NC>(f, off, omega_r);
}

#ifndef SS_WARP_TRIG
#define SS_WARP_TRIG 1        // warp-shared per-interval sincos (warp_trig); 0: every lane evaluates its own
#endif
#ifndef SS_WARP_TRIG_EXIT
#define SS_WARP_TRIG_EXIT 1   // include a8's exit angle (held through the step loop) in the shared set
#endif
// The frame exit's sincos (a8), when warp_trig supplied it.
struct ExitTrig {
  bool pre;
  double s, c;
};

// Per-interval trigonometry shared across a warp.  An interval's prologue takes seven sincos whose arguments depend
// only on the sweep and on ω_r — the field's RF rotations ω·g1δt, ω·g2δt, ω·δt (init_cf4), the frame's ω_r·g1δt,
// ω_r·g2δt, ω_r·δt and the exit angle of a8 — and ω_r is the same for every interval outside a pulse window.  When
// all 32 lanes hold the same sweep and ω_r (a warp-uniform test), lane j evaluates the j-th of them and the warp
// exchanges the results by shuffles: one sincos latency per warp instead of seven in a row (the ncu source view put
// these calls at ≈ 10 % of the C3 kernel's warp samples).  Same expressions, same library sincos: bit-identical values.
template <class FLD>
__device__ __forceinline__ bool warp_trig(const FLD& fld, int64_t b, double omega_r, double exit_angle,
                                          const IntervalParams& prm, double tr[14]) {
  if (__activemask() != 0xffffffffu) return false;
  const long long b0 = __shfl_sync(0xffffffffu, (long long)b, 0);
  const double w0 = __shfl_sync(0xffffffffu, omega_r, 0);
  if (!__all_sync(0xffffffffu, (long long)b == b0 && omega_r == w0)) return false;
  const int lane = threadIdx.x & 31;
  const double W = fld.rf();
  double x = 0.0;
  switch (lane) {
    case 0: x = W * prm.g1dt; break;
    case 1: x = W * prm.g2dt; break;
    case 2: x = W * prm.dt; break;
    case 3: x = omega_r * prm.g1dt; break;
    case 4: x = omega_r * prm.g2dt; break;
    case 5: x = omega_r * prm.dt; break;
    case 6: x = exit_angle; break;
  }
  double sn, cs;
  sincos(x, &sn, &cs);
#pragma unroll
  for (int j = 0; j < 7; ++j) {
    tr[2 * j] = __shfl_sync(0xffffffffu, sn, j);
    tr[2 * j + 1] = __shfl_sync(0xffffffffu, cs, j);
  }
  return true;
}

// Rows a1–a7 for fine steps [l_begin, l_end) of interval k of sweep b: A = the product of those steps' exponentials
// minus I, in the rotating frame at ω_r (residual form, reading R9) — the whole interval's U_r − I when the range is
// [0, L), else a piece that the caller multiplies with its neighbours' (same samples, same frame).
template <int SPIN, int EXPO, int METHOD, int FIELD, typename T>
__device__ __forceinline__ void interval_residual(const IntervalParams& prm, int64_t b, int64_t k, int64_t l_begin,
                                                  int64_t l_end, Res<AccDim<SPIN, EXPO>::D, T>& A_out,
                                                  double& omega_r_out, ExitTrig& ex) {
  constexpr int D = SpinDim<SPIN>::D;
  constexpr int P = FieldParams<FIELD>::P;
  constexpr int NC = NumCoeffs<EXPO>::N;             // 4, or 8 for the general spin-one exponentiator
  (void)D;

  double p[P];
#pragma unroll
  for (int j = 0; j < P; ++j) p[j] = __ldg(prm.sweep + b * P + j);

  // a1: t_k = fl(t0 + fl(k·Δt)) (reading R7); ω_r from the lab field at the interval midpoint.
  const double t_k = __dadd_rn(prm.t0, __dmul_rn((double)k, prm.dt_out));
  Field<FIELD> fld;
  fld.init(p, t_k);
  double omega_r = 0.0;
  if (prm.frame) {
    double f[8];
    fld.sample(prm.half_dt_out, f);
    omega_r = f[2];
  }

  FrameCF4 frame2;
  ex.pre = false;
  if (METHOD == CF4) {
    // a8's angle: ω_rΔt/2 for the SU(2) forms (spin-half, compact operators), ω_rΔt for dense spin-one (make_op)
    const double exit_angle = (D == 2 || prm.op_format == OP_SU2) ? 0.5 * omega_r * prm.dt_out : omega_r * prm.dt_out;
    double tr[14];
    if (SS_WARP_TRIG && warp_trig(fld, b, omega_r, exit_angle, prm, tr)) {
      fld.init_cf4_pre(tr);
      frame2.init_pre(omega_r, tr + 6);
      if (SS_WARP_TRIG_EXIT) {
        ex.pre = true;
        ex.s = tr[12];
        ex.c = tr[13];
      }
    } else {
      fld.init_cf4(prm.g1dt, prm.g2dt, prm.dt);
      frame2.init(omega_r, prm.g1dt, prm.g2dt, prm.dt);
    }
  }

  constexpr int DA = AccDim<SPIN, EXPO>::D;         // accumulated residual: SU(2) form (2) or dense 3×3
  // SU(2) closed form: |a| ≤ (|w+| + |w−|)·|f| (CF4) or δt·|f| ≤ 2^-13 on every step of this interval ⇒ short series
  int su2_ser = 0;
  if constexpr (DA == 2 && sizeof(T) == 8) {
    const double rb = (METHOD == CF4 ? fabs(prm.wpd) + fabs(prm.wmd) : prm.dt) * field_bound(fld, omega_r, 0);
    // 2^-13 / 2^-7 with a margin for the rounding of a and of the bound (expo_su2's short / medium series)
    su2_ser = rb * 1.01 <= 1.220703125e-04 ? 2 : (rb * 1.01 <= 0.0078125 ? 1 : 0);
  }
  Res<DA, T> A;   // U_r − I, U_r initialised to the identity
  res_zero(A);

  // One fine step.  ANCHOR (exact sincos of the phase steppers, every kAnchor-th step) and PULSE (this interval can
  // meet the neural field's pulse window) are compile-time, so the step body carries no per-step branches for them.
  auto step = [&](int64_t l, auto anchor_c, auto pulse_c, auto short_c) {
    const bool ANCHOR = anchor_c.value, PULSE = pulse_c.value;   // compile-time for BoolC, run-time for RtBool
    const int SER = short_c.value;
    const double base = __dmul_rn((double)l, prm.dt);
    Res<DA, T> u;
    if (METHOD == CF4) {
      // a2/a3: samples at t_k + (l + g1,2)δt, rotated into the frame.
      double f1[NC], f2[NC];
#pragma unroll
      for (int j = 4; j < NC; ++j) f1[j] = f2[j] = 0.0;   // 4-coefficient fields under the su(3) exponentiator
      // exact sincos on anchor steps, rotation by e^{iωδt} in between (measured: +1.4 % on spin-one C3 despite
      // a few extra spill slots outside the squaring loops, +70 % on trig-bound spin-half)
      fld.sample_cf4(base, ANCHOR, PULSE, __dadd_rn(base, prm.g1dt), __dadd_rn(base, prm.g2dt), f1, f2);
      if (prm.frame) frame2.apply<NC, zero_y_of<Field<FIELD>>(nullptr)>(base, ANCHOR, f1, f2);
      // a4: H̄1 δt = (w+ f1 + w− f2) δt, H̄2 δt = (w− f1 + w+ f2) δt (Eqs. cf4_sample_1/2), δt folded into w±.
      T a1[NC], a2[NC];
#pragma unroll
      for (int j = 0; j < NC; ++j) {
        a1[j] = (T)fma(prm.wpd, f1[j], prm.wmd * f2[j]);
        a2[j] = (T)fma(prm.wmd, f1[j], prm.wpd * f2[j]);
      }
      if constexpr (SPIN == SPIN_ONE && EXPO == EXP_LIE_TROTTER && sizeof(T) == 4) {
        // FP32 mode: both exponentials' symmetric squarings in lockstep, packed one per float2 lane (FFMA2)
        Sym3<float> m1, m2;
        float c1, s1, c2, s2;
        trotter_init<float>(a1, prm.tau, m1, c1, s1);
        trotter_init<float>(a2, prm.tau, m2, c2, s2);
        Sym3<float2> m = sym_pack(m1, m2);
#pragma unroll 2
        for (int it = 0; it < prm.tau; ++it) lt_square<float2>(m);
        sym_unpack(m, m1, m2);
        Res<D, T> e;
        trotter_expand<T>(m1, c1, s1, e);
        res_mul(e, A, u);
        trotter_expand<T>(m2, c2, s2, e);
        res_mul(e, u, A);
        return;
      }
      if constexpr (SPIN == SPIN_ONE && EXPO == EXP_LIE_TROTTER_SU3 && sizeof(T) == 4) {
        // FP32 mode, general spin-one: the same lockstep squarings on the tridiagonalised factors (reading R20)
        Sym3<float> m1, m2;
        Su3W<float> w1, w2;
        su3_init<float>(a1, prm.tau, m1, w1);
        su3_init<float>(a2, prm.tau, m2, w2);
        Sym3<float2> m = sym_pack(m1, m2);
#pragma unroll 2
        for (int it = 0; it < prm.tau; ++it) lt_square<float2>(m);
        sym_unpack(m, m1, m2);
        Res<D, T> e;
        su3_expand<T>(m1, w1, e);
        res_mul(e, A, u);
        su3_expand<T>(m2, w2, e);
        res_mul(e, u, A);
        return;
      }
      // a5/a6/a7: u·U_r = e2·(e1·U_r) (Eq. cf4_implementation), folded one exponential at a time so only
      // one exponential is live in registers (occupancy).  Residual form: A ← e + A + e·A.
      {
        Res<DA, T> e;
        Expo<SPIN, EXPO, T>::run(a1, prm.tau, e, SER);
        res_mul(e, A, u);
      }
      {
        Res<DA, T> e;
        Expo<SPIN, EXPO, T>::run(a2, prm.tau, e, SER);
        res_mul(e, u, A);
      }
      return;
    } else {
      double f[NC];
#pragma unroll
      for (int j = 4; j < NC; ++j) f[j] = 0.0;
      if (METHOD == MIDPOINT) {                       // one sample at t + δt/2 (reading R13)
        sample_in_frame<NC>(fld, __dadd_rn(base, prm.half_dt), omega_r, prm.frame, f);
      } else {                                        // HEUN: average of t and t + δt
        double fa[NC], fb[NC];
#pragma unroll
        for (int j = 4; j < NC; ++j) fa[j] = fb[j] = 0.0;
        sample_in_frame<NC>(fld, base, omega_r, prm.frame, fa);
        sample_in_frame<NC>(fld, __dmul_rn((double)(l + 1), prm.dt), omega_r, prm.frame, fb);
#pragma unroll
        for (int j = 0; j < NC; ++j) f[j] = 0.5 * (fa[j] + fb[j]);
      }
      T a[NC];
#pragma unroll
      for (int j = 0; j < NC; ++j) a[j] = (T)(f[j] * prm.dt);
      Expo<SPIN, EXPO, T>::run(a, prm.tau, u, SER);
    }
    // a7: U_r ← u·U_r, residual form: A ← u + A + u·A.
    Res<DA, T> An;
    res_mul(u, A, An);
    A = An;
  };
  auto run_steps = [&](auto pulse_c, auto short_c) {
#pragma unroll 1
    for (int64_t l0 = l_begin; l0 < l_end; l0 += kAnchor) {
      step(l0, BoolC<true>{}, pulse_c, short_c);
      const int64_t l1 = l0 + kAnchor < l_end ? l0 + kAnchor : l_end;
      SS_UNROLL(SS_STEP_UNROLL)
      for (int64_t l = l0 + 1; l < l1; ++l) step(l, BoolC<false>{}, pulse_c, short_c);
    }
  };
  if constexpr (DA == 2) {
    // spin-half / analytic spin-one (short, trig-heavy steps): specialised bodies, C4 1.05e11 → 1.24e11 fine steps/s;
    // the short-series choice too (SS_SU2_SHORT_BODIES)
    auto with_pulse = [&](auto pulse_c) {
      if constexpr (SS_SU2_SHORT_BODIES && sizeof(T) == 8) {
        if (su2_ser == 2) run_steps(pulse_c, IntC<2>{});
        else if (su2_ser == 1) run_steps(pulse_c, IntC<1>{});
        else run_steps(pulse_c, IntC<0>{});
      } else {
        run_steps(pulse_c, RtInt{su2_ser});
      }
    };
    if (field_pulse_possible(fld, prm.dt_out, 0)) with_pulse(BoolC<true>{});
    else with_pulse(BoolC<false>{});
  } else {
    // 3×3 paths: groups of kAnchor steps, the first an anchor step — two step bodies (anchor, rotated) with the
    // pulse test at run time (round 1's four (anchor × pulse) bodies spilled more and cost C3 2.5 %; this pair: +0.3 %,
    // profiles/r02/s27_anch/)
#pragma unroll 1
    for (int64_t l0 = l_begin; l0 < l_end; l0 += kAnchor) {
      step(l0, BoolC<true>{}, BoolC<true>{}, IntC<0>{});
      const int64_t l1 = l0 + kAnchor < l_end ? l0 + kAnchor : l_end;
#pragma unroll 1
      for (int64_t l = l0 + 1; l < l1; ++l) step(l, BoolC<false>{}, BoolC<true>{}, IntC<0>{});
    }
  }

  A_out = A;
  omega_r_out = omega_r;
}

// a8: U_k = R_{ω_r}(−Δt)(I + A) = diag(e^{−iω_r m Δt})(I + A), as the dense D×D complex matrix ...
template <int D, int DA, typename T>
__device__ __forceinline__ void make_op(const Res<DA, T>& A, double omega_r, const ExitTrig& ex,
                                        const IntervalParams& prm, CM<D>& m) {
  double ph_re[D], ph_im[D];
  {
    double s, c;
    if (ex.pre) { s = ex.s; c = ex.c; }
    else if (D == 2) sincos(0.5 * omega_r * prm.dt_out, &s, &c);
    else sincos(omega_r * prm.dt_out, &s, &c);
    ph_re[0] = c; ph_im[0] = -s;                      // m = +1 (or +½)
    ph_re[D - 1] = c; ph_im[D - 1] = s;               // m = −1 (or −½)
    if (D == 3) { ph_re[1] = 1.0; ph_im[1] = 0.0; }   // m = 0
  }
  Res<D, T> Ad;                                      // D¹ map of the SU(2) accumulator (analytic spin-one)
  acc_to_dim<T>(A, Ad);
#pragma unroll
  for (int r = 0; r < D; ++r)
#pragma unroll
    for (int cc = 0; cc < D; ++cc) {
      const double mr = (double)res_re(Ad, r, cc) + (r == cc ? 1.0 : 0.0);
      const double mi = (double)res_im(Ad, r, cc);
      m.re[r * D + cc] = ph_re[r] * mr - ph_im[r] * mi;
      m.im[r * D + cc] = ph_re[r] * mi + ph_im[r] * mr;
    }
}
// ... or (SU(2)-form accumulators) compact: the SU(2) element (a, b) = e^{−iω_rΔt/2}·(1 + δa, b) — R(−Δt) is
// diag(p, p*) with p = e^{−iω_rΔt/2} in SU(2), and D¹ of it for the analytic spin-one path (diag(p², 1, p*²)).
template <int D, typename T>
__device__ __forceinline__ void make_op(const Res<2, T>& A, double omega_r, const ExitTrig& ex,
                                        const IntervalParams& prm, SU<D>& u) {
  double s, c;
  if (ex.pre) { s = ex.s; c = ex.c; }
  else sincos(0.5 * omega_r * prm.dt_out, &s, &c);
  const double ar = 1.0 + (double)A.ar, ai = (double)A.ai, br = (double)A.br, bi = (double)A.bi;
  u.ar = c * ar + s * ai; u.ai = c * ai - s * ar;     // (c − is)(ar + i ai)
  u.br = c * br + s * bi; u.bi = c * bi - s * br;
}

// Fused path (DESIGN.md §5 item 16; SURVEY §8(a) a9 "Fusion"): this thread owns the n ≤ ipt consecutive intervals
// [k_lo, k_lo + n) of sweep b, writes each U_k and folds it into the run product G ← U_k·G (later·earlier),
// held in shared memory (the kernels sit at their register budget), then writes G to run_agg[slot].
template <class M>
__device__ __forceinline__ void run_fold(double2* acc, const M& op, double2* dst) {
  M g;
  cm_load(acc, g);
  cm_store(acc, cm_mul(op, g));
  cm_store(dst, op);
}
template <int SPIN, int EXPO, int METHOD, int FIELD, typename T>
__device__ __forceinline__ void interval_run(const IntervalParams& prm, int64_t b, int64_t k_lo, int64_t n,
                                             int64_t slot) {
  constexpr int D = SpinDim<SPIN>::D, DA = AccDim<SPIN, EXPO>::D;
  // the operator format is a run-time choice, but the step loop (interval_residual) appears once in the code: only
  // the small per-interval fold is specialised per format (two inlined copies of the loop bodies defeated inlining)
  [[maybe_unused]] const bool su = DA == 2 && prm.op_format == OP_SU2;
  extern __shared__ __align__(16) double2 ss_run_smem[];
  double2* acc = ss_run_smem + threadIdx.x * (D * D);
  if (DA == 2 && su) { SU<D> e; cm_eye(e); cm_store(acc, e); }
  else { CM<D> e; cm_eye(e); cm_store(acc, e); }
  double2* U = reinterpret_cast<double2*>(prm.unitaries);
#pragma unroll 1
  for (int64_t j = 0; j < n; ++j) {
    Res<DA, T> A;
    double omega_r;
    ExitTrig ex;
    interval_residual<SPIN, EXPO, METHOD, FIELD, T>(prm, b, prm.k_begin + k_lo + j, 0, prm.L, A, omega_r, ex);
    const int64_t i = b * prm.k_count + k_lo + j;
    if constexpr (DA == 2) {
      if (su) {
        SU<D> op;
        make_op(A, omega_r, ex, prm, op);
        run_fold(acc, op, U + i * 2);
        continue;
      }
    }
    CM<D> op;
    make_op(A, omega_r, ex, prm, op);
    run_fold(acc, op, U + i * (D * D));
  }
  if constexpr (DA == 2) {
    if (su) {
      SU<D> g;
      cm_load(acc, g);
      cm_store(reinterpret_cast<double2*>(prm.run_agg) + slot * 2, g);
      return;
    }
  }
  CM<D> g;
  cm_load(acc, g);
  cm_store(reinterpret_cast<double2*>(prm.run_agg) + slot * (D * D), g);
}

// U_k of the launch's flat interval index i (sweep-major) from the residual A of the whole interval, in the output
// format: dense D×D, or compact SU(2) for the SU(2)-form accumulators.
template <int D, int DA, typename T>
__device__ __forceinline__ void store_op(const IntervalParams& prm, const Res<DA, T>& A, double omega_r,
                                         const ExitTrig& ex, int64_t i) {
  if constexpr (DA == 2) {
    if (prm.op_format == OP_SU2) {
      SU<D> u;
      make_op(A, omega_r, ex, prm, u);
      cm_store(reinterpret_cast<double2*>(prm.unitaries) + i * 2, u);
      return;
    }
  }
  CM<D> m;
  make_op(A, omega_r, ex, prm, m);
  cm_store(reinterpret_cast<double2*>(prm.unitaries) + i * (D * D), m);
}

// Kernel modes (separate instances, so each one's code is untouched by the other):
//   MODE_SPLIT: one interval per S lanes (S = 1: per thread; S > 1: the sub-interval split, DESIGN.md §5 item 8);
//   MODE_FUSED: prm.run_agg is set, S = 1, thread slot gt of sweep b owns ipt intervals (§5 item 16).
enum { MODE_SPLIT = 0, MODE_FUSED = 1 };

template <int SPIN, int EXPO, int METHOD, int FIELD, typename T, int MODE>
__device__ __forceinline__ void interval_body(const IntervalParams& prm) {
  constexpr int D = SpinDim<SPIN>::D;
  constexpr int DA = AccDim<SPIN, EXPO>::D;
  const int64_t gt = (int64_t)blockIdx.x * kIntervalThreads + threadIdx.x;
  if constexpr (MODE == MODE_FUSED) {
    const int64_t b = gt / prm.k_stride, t = gt - b * prm.k_stride;
    if (b >= prm.batch) return;
    const int64_t k_lo = t * prm.ipt, n = min(prm.ipt, prm.k_count - k_lo);
    interval_run<SPIN, EXPO, METHOD, FIELD, T>(prm, b, k_lo, n, gt);
    return;
  } else {
    const int S = prm.split;
    const int64_t i = gt / S;                        // interval index (sweep-major)
    const int part = (int)(gt - i * S);
    const bool active = i < prm.n_threads;
    if (S == 1 && !active) return;                   // with S > 1 every lane must reach the shuffles
    const int64_t ic = active ? i : 0;
    const int64_t b = ic / prm.k_count;
    const int64_t k = prm.k_begin + (ic - b * prm.k_count);
    const int64_t l_begin = (prm.L * part) / S, l_end = active ? (prm.L * (part + 1)) / S : l_begin;
    Res<DA, T> A;
    double omega_r;
    ExitTrig ex;
    interval_residual<SPIN, EXPO, METHOD, FIELD, T>(prm, b, k, l_begin, l_end, A, omega_r, ex);
    // Sub-interval split: lane p holds the partial product of its fine steps; combine later·earlier in a shuffle tree
    // (U_r = P_{S−1} ⋯ P_0, same samples, only the association of the product differs).
    if (S > 1) {
      for (int off = 1; off < S; off <<= 1) {
        const Res<DA, T> B = res_shfl_down(A, off);
        if ((part & (2 * off - 1)) == 0) {
          Res<DA, T> C;
          res_mul(B, A, C);
          A = C;
        }
      }
    }
    if (part != 0 || !active) return;
    store_op<D>(prm, A, omega_r, ex, i);
  }
}

template <int SPIN, int EXPO, int METHOD, int FIELD, typename T, int MODE>
__global__ void __launch_bounds__(kIntervalThreads, kIntervalMinBlocks<SPIN, EXPO, T>())
interval_kernel(const IntervalParams prm) {
  interval_body<SPIN, EXPO, METHOD, FIELD, T, MODE>(prm);
}

#ifndef __CUDACC_RTC__
// Dynamic shared memory of an interval launch: the fused path's per-thread run product (≤ 9 complex128).
inline size_t interval_smem(const IntervalParams& prm) {
  return prm.run_agg ? (size_t)kIntervalThreads * 9 * 16 : 0;
}

// Blocks of an interval launch: one lane per interval slot (S lanes per interval with the split).
inline int64_t interval_blocks(const IntervalParams& prm) {
  return (prm.n_threads * prm.split + kIntervalThreads - 1) / kIntervalThreads;
}

template <int SPIN, int EXPO, int METHOD, int FIELD, typename T>
cudaError_t launch_interval(const IntervalParams& prm, cudaStream_t stream) {
  const int64_t blocks = interval_blocks(prm);
  if (blocks <= 0) return cudaSuccess;
  if (prm.run_agg)
    interval_kernel<SPIN, EXPO, METHOD, FIELD, T, MODE_FUSED><<<(unsigned)blocks, kIntervalThreads, interval_smem(prm), stream>>>(prm);
  else
    interval_kernel<SPIN, EXPO, METHOD, FIELD, T, MODE_SPLIT><<<(unsigned)blocks, kIntervalThreads, 0, stream>>>(prm);
  return cudaGetLastError();
}
#endif  // !__CUDACC_RTC__

// ---- advisory Magnus-convergence diagnostic --------------------------------------------------
// The Magnus series of a step converges if ∫‖H‖₂ over it < ξ ≈ 1.08686870.  For every fine step this estimates
// the integral by the two-point Gauss–Legendre rule on the CF4 sample times, δt·(‖H(t₁)‖₂ + ‖H(t₂)‖₂)/2, in the frame
// the integrator uses, and out[b] = the maximum over sweep b (atomic max on the non-negative doubles' bit patterns).
// ‖H‖₂ is exact: |ω|/2 for spin-half; for spin-one the largest |eigenvalue| of the traceless Hermitian 3×3 from the
// roots of λ³ − pλ − q (p = tr H²/2, q = det H) in trigonometric form.
template <int SPIN, int NC> __device__ __forceinline__ double spectral_norm(const double* f) {
  if constexpr (SPIN == SPIN_HALF) {
    return 0.5 * sqrt(fma(f[0], f[0], fma(f[1], f[1], f[2] * f[2])));
  } else {
    const double d0 = f[2] + f[3] * kThird, d1 = -2.0 * f[3] * kThird, d2 = f[3] * kThird - f[2];
    double ur = 0.0, ui = 0.0, vr = 0.0, vi = 0.0;
    if constexpr (NC == 8) { ur = f[4]; ui = -f[5]; vr = f[6]; vi = -f[7]; }
    const double ar = (f[0] + vr) * kRsqrt2, ai = (-f[1] + vi) * kRsqrt2;      // H01
    const double br = (f[0] - vr) * kRsqrt2, bi = (-f[1] - vi) * kRsqrt2;      // H12
    const double na = ar * ar + ai * ai, nb = br * br + bi * bi, ng = ur * ur + ui * ui;   // |H01|², |H12|², |H02|²
    const double p = 0.5 * (d0 * d0 + d1 * d1 + d2 * d2) + na + nb + ng;
    // det H = d0 d1 d2 + 2 Re(H01 H12 conj(H02)) − d0|H12|² − d1|H02|² − d2|H01|²
    const double pr = ar * br - ai * bi, pim = ar * bi + ai * br;
    const double q = d0 * d1 * d2 + 2.0 * (pr * ur + pim * ui) - d0 * nb - d1 * ng - d2 * na;
    if (!(p > 0.0)) return 0.0;
    const double r = 2.0 * sqrt(p / 3.0);
    double c = 1.5 * q / p * sqrt(3.0 / p);
    c = fmin(1.0, fmax(-1.0, c));
    const double phi = acos(c) / 3.0;
    const double l0 = r * cos(phi), l2 = r * cos(phi + 2.0943951023931957);   // largest and smallest eigenvalues
    return fmax(fabs(l0), fabs(l2));
  }
}

template <int SPIN, int EXPO, int FIELD>
__device__ __forceinline__ void magnus_body(const IntervalParams& prm, double* out) {
  constexpr int P = FieldParams<FIELD>::P;
  constexpr int NC = NumCoeffs<EXPO>::N;
  const int64_t i = (int64_t)blockIdx.x * 128 + threadIdx.x;
  if (i >= prm.n_threads) return;
  const int64_t b = i / prm.k_count;
  const int64_t k = prm.k_begin + (i - b * prm.k_count);
  double p[P];
#pragma unroll
  for (int j = 0; j < P; ++j) p[j] = __ldg(prm.sweep + b * P + j);
  const double t_k = __dadd_rn(prm.t0, __dmul_rn((double)k, prm.dt_out));
  Field<FIELD> fld;
  fld.init(p, t_k);
  double omega_r = 0.0;
  if (prm.frame) {
    double f[8];
    fld.sample(prm.half_dt_out, f);
    omega_r = f[2];
  }
  double m = 0.0;
  for (int64_t l = 0; l < prm.L; ++l) {
    const double base = __dmul_rn((double)l, prm.dt);
    double f1[8] = {0, 0, 0, 0, 0, 0, 0, 0}, f2[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    sample_in_frame<NC>(fld, __dadd_rn(base, prm.g1dt), omega_r, prm.frame, f1);
    sample_in_frame<NC>(fld, __dadd_rn(base, prm.g2dt), omega_r, prm.frame, f2);
    m = fmax(m, 0.5 * prm.dt * (spectral_norm<SPIN, NC>(f1) + spectral_norm<SPIN, NC>(f2)));
  }
  atomicMax(reinterpret_cast<unsigned long long*>(out) + b, (unsigned long long)__double_as_longlong(m));
}

template <int SPIN, int EXPO, int FIELD>
__global__ void __launch_bounds__(128) magnus_kernel(const IntervalParams prm, double* out) {
  magnus_body<SPIN, EXPO, FIELD>(prm, out);
}

#ifndef __CUDACC_RTC__
template <int SPIN, int EXPO, int FIELD>
cudaError_t launch_magnus(const IntervalParams& prm, double* out, cudaStream_t stream) {
  const int64_t blocks = (prm.n_threads + 127) / 128;
  if (blocks <= 0) return cudaSuccess;
  magnus_kernel<SPIN, EXPO, FIELD><<<(unsigned)blocks, 128, 0, stream>>>(prm, out);
  return cudaGetLastError();
}
#endif

#ifndef __CUDACC_RTC__
// Small kernel for element-wise parity of the exponentiators (ss_exponentiate).
template <int SPIN, int EXPO, typename T>
__global__ void exponentiate_kernel(int64_t n, const double* args, int tau, double* out) {
  constexpr int D = SpinDim<SPIN>::D;
  constexpr int NA = NumCoeffs<EXPO>::N;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  T a[NA];
#pragma unroll
  for (int j = 0; j < NA; ++j) a[j] = (T)args[NA * i + j];
  Res<AccDim<SPIN, EXPO>::D, T> e0;
  Expo<SPIN, EXPO, T>::run(a, tau, e0);
  Res<D, T> e;
  acc_to_dim<T>(e0, e);
  double2* o = reinterpret_cast<double2*>(out) + i * D * D;
#pragma unroll
  for (int r = 0; r < D; ++r)
#pragma unroll
    for (int c = 0; c < D; ++c)
      o[r * D + c] = make_double2((double)res_re(e, r, c) + (r == c ? 1.0 : 0.0), (double)res_im(e, r, c));
}

template <int SPIN, int EXPO, typename T>
cudaError_t launch_exponentiate(int64_t n, const double* args, int tau, double* out, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  exponentiate_kernel<SPIN, EXPO, T><<<(unsigned)((n + 127) / 128), 128, 0, stream>>>(n, args, tau, out);
  return cudaGetLastError();
}
#endif  // !__CUDACC_RTC__

}  // namespace ssb
