// spinsim_device.cuh — device math of the Spinsim hot path for sm_100a (rows a1–a8 of SURVEY §8(a)).
//
// Everything is header-only __device__ __forceinline__ code, templated on the stepper real type T (double for the
// FP64 path, float for the FP32 mode).  Time, phases, field samples and the frame angle are always FP64
// (FP32 mode).  No tensor cores: the operands are 2×2 / 3×3 complex matrices held in registers.
//
// Residual representation: a matrix M close to the identity is carried as a = M − I; products use
// (I+a)(I+b) − I = a + b + ab and squares (I+a)² − I = (a + 2I)a, so the accumulated interval unitary never suffers
// the cancellation of subtracting 1 from near-unity diagonals (reading R9).
#pragma once

#ifndef __CUDACC_RTC__
#include <cuda_runtime.h>
#include <stdint.h>
#else   // NVRTC compile of a user field (user_field.cu): no system headers
typedef long long int64_t;
typedef int int32_t;
typedef unsigned int uint32_t;
typedef unsigned long long uint64_t;
#endif

namespace ssb {

enum { SPIN_HALF = 1, SPIN_ONE = 2 };
enum { CF4 = 0, MIDPOINT = 1, HEUN = 2 };
enum { EXP_ANALYTIC = 0, EXP_LIE_TROTTER = 1, EXP_LIE_TROTTER_SU3 = 2 };
enum { FIELD_CONSTANT = 0, FIELD_RABI_LINEAR = 1, FIELD_RABI_CIRCULAR = 2, FIELD_NEURAL = 3, FIELD_GRADIENT = 4,
       FIELD_USER = 5, FIELD_SU3_CONSTANT = 6, FIELD_SU3_DRIVE = 7 };

// Number of Hamiltonian coefficients a field sample carries for an exponentiator: 4 (ωx, ωy, ωz, ωq)
// or 8 for the general spin-one exponentiator (+ ωu1, ωu2, ωv1, ωv2, reading R19).
template <int EXPO> struct NumCoeffs { static constexpr int N = (EXPO == EXP_LIE_TROTTER_SU3) ? 8 : 4; };

// ---- constants: correctly rounded doubles (reading R7) ------------------------------------------------
constexpr double kG1 = 0x1.b0cb174df99c7p-3;       // ½(1 − 1/√3)  Gauss–Legendre node
constexpr double kG2 = 0x1.93cd3a2c8198ep-1;       // ½(1 + 1/√3)
constexpr double kWPlus = 0x1.13cd3a2c8198ep-1;    // (3 + 2√3)/12 (Eq. cf4_sample_1)
constexpr double kWMinus = -0x1.3cd3a2c8198e2p-5;  // (3 − 2√3)/12 (negative)
constexpr double kTwoPi1 = 0x1.921fb54442d18p+2;   // 2π = kTwoPi1 + kTwoPi2 + kTwoPi3 (Cody–Waite, reading R8)
constexpr double kTwoPi2 = 0x1.1a62633145c07p-52;
constexpr double kTwoPi3 = -0x1.f1976b7ed8fbcp-108;
constexpr double kInvTwoPi = 0x1.45f306dc9c883p-3;
constexpr double kRsqrt2 = 0x1.6a09e667f3bcdp-1;   // 1/√2
constexpr double kSqrt2 = 0x1.6a09e667f3bcdp+0;
constexpr double kThird = 0x1.5555555555555p-2;

// Format of the interval operators handed from the interval kernel to the state scan: the dense dim×dim complex
// matrix (the public U_k layout), or — for the SU(2)-form paths when U_k is not an output — the SU(2) element (a, b)
// of U = [[a, b], [−b*, a*]] (2 complex128 per interval; D¹ of it for the analytic spin-one path, reading R14).
enum { OP_DENSE = 0, OP_SU2 = 1 };

template <int SPIN> struct SpinDim { static constexpr int D = (SPIN == SPIN_HALF) ? 2 : 3; };
template <int F> struct FieldParams;
template <> struct FieldParams<FIELD_CONSTANT> { static constexpr int P = 4; };
template <> struct FieldParams<FIELD_RABI_LINEAR> { static constexpr int P = 2; };
template <> struct FieldParams<FIELD_RABI_CIRCULAR> { static constexpr int P = 2; };
template <> struct FieldParams<FIELD_NEURAL> { static constexpr int P = 7; };
template <> struct FieldParams<FIELD_GRADIENT> { static constexpr int P = 2; };
template <> struct FieldParams<FIELD_SU3_CONSTANT> { static constexpr int P = 8; };
template <> struct FieldParams<FIELD_SU3_DRIVE> { static constexpr int P = 6; };

// Series coefficients of cos(r/2) − 1 (÷ r², highest first) and sin(r/2)/r (highest first), constant bank.
__constant__ double kSu2Series[10] = {-1.0 / 3715891200.0, 1.0 / 10321920.0, -1.0 / 46080.0, 1.0 / 384.0, -0.125,
                                      1.0 / 185794560.0, -1.0 / 645120.0, 1.0 / 3840.0, -1.0 / 48.0, 0.5};

// ---- precision-generic scalar helpers ---------------------------------------------------------------------------
__device__ __forceinline__ double fmaT(double a, double b, double c) { return fma(a, b, c); }
__device__ __forceinline__ float fmaT(float a, float b, float c) { return fmaf(a, b, c); }
// float2 = two independent FP32 lanes (the FP32 mode runs both CF4 exponentials of a step in lockstep, one per lane):
// Blackwell's packed FFMA2 / FMUL2 / FADD2, with negations folded into the operands by ptxas.
__device__ __forceinline__ float2 fmaT(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 operator*(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 operator+(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 operator-(float2 a) { return make_float2(-a.x, -a.y); }
template <typename T> __device__ __forceinline__ T splat(double v) { return T(v); }
template <> __device__ __forceinline__ float2 splat<float2>(double v) { return make_float2((float)v, (float)v); }
__device__ __forceinline__ void sincosT(double x, double* s, double* c) { sincos(x, s, c); }
__device__ __forceinline__ void sincosT(float x, float* s, float* c) { sincosf(x, s, c); }
__device__ __forceinline__ double sqrtT(double x) { return sqrt(x); }
__device__ __forceinline__ float sqrtT(float x) { return sqrtf(x); }
__device__ __forceinline__ double rsqrtT(double x) { return rsqrt(x); }
__device__ __forceinline__ float rsqrtT(float x) { return rsqrtf(x); }

// sin/cos of a small angle (|x| ≤ 2^-6) by its Taylor polynomial through x^9 / x^8 (truncation < 1e-25 relative):
// the Lie–Trotter arguments are Φ/2, θ/2 divided by n = 2^τ, so this path is the common one; larger arguments go to
// the library sincos.
template <typename T> __device__ __forceinline__ void sincos_small(T x, T* s, T* c) {
  const T x2 = x * x;
  *s = fmaT(x * x2, fmaT(x2, fmaT(x2, fmaT(x2, T(1.0 / 362880.0), T(-1.0 / 5040.0)), T(1.0 / 120.0)), T(-1.0 / 6.0)), x);
  *c = fmaT(x2, fmaT(x2, fmaT(x2, fmaT(x2, T(1.0 / 40320.0), T(-1.0 / 720.0)), T(1.0 / 24.0)), T(-0.5)), T(1));
}

template <typename T> __device__ __forceinline__ void sincos_tiny(T x, T* s, T* c) {
  const T x2 = x * x;
  *s = fmaT(x * x2, T(-1.0 / 6.0), x);
  *c = fmaT(x2, T(-0.5), T(1));
}

// Reduce ω·t (both FP64) to (−π, π] accurately: exact product as hi + lo (FMA), then Cody–Waite with a 3-part 2π.
// Never a single-double 2π (SURVEY [V15]).  |result error| ≲ 5e-16 for |ω t| ≲ 1e9.
__device__ __forceinline__ double reduce_phase(double w, double t) {
  const double hi = __dmul_rn(w, t);
  const double lo = fma(w, t, -hi);
  const double n = rint(hi * kInvTwoPi);
  double r = fma(-n, kTwoPi1, hi);
  r = fma(-n, kTwoPi2, r);
  r = fma(-n, kTwoPi3, r);
  return r + lo;
}

// ---- built-in field functions (Eq. neural_pulse; MRI example P:668-669) ------------------------
// A field object is initialised once per interval with its sweep parameters and t_k; sample(off) returns
// (ωx, ωy, ωz, ωq) at time t_k + off (the (t_k, off) pair is never rounded to one double — reading R8).
template <int F> struct Field;

// e^{i(ph0 + w·base_l)} along the fine steps of one interval: an exact sincos on anchor steps (every kAnchor-th step
// of a lane, and its first), otherwise advanced by the per-interval rotation e^{iwδt} (error ≲ kAnchor·2 ulp of a
// unit vector, ≲ 7e-15 rad at kAnchor = 32; the grid's base_l = fl(l·δt) differs from l·δt by < 1 ulp, i.e.
// ≲ 1e-15 rad at |w δt| ≤ 5).  Anchors every 8 / 16 / 32 / 64 steps (profiles/r02/s13_anchor/): C4 1.50 / 1.57 / 1.61 /
// 1.63e11 fine steps/s, C5 analytic 1.248 / 1.187 / 1.188 ms, the 3×3 paths unchanged (their L = 10 intervals anchor
// once); parity unchanged (the C4 every-state check passes at 64).
#ifndef SS_ANCHOR
#define SS_ANCHOR 32
#endif

constexpr int kAnchor = SS_ANCHOR;
struct PhaseStepper {
  double w, ph0, cd, sd, c, s;
  __device__ __forceinline__ void init(double w_, double ph0_, double dt) {
    w = w_; ph0 = ph0_;
    sincos(w * dt, &sd, &cd);
  }
  // the same with sincos(w·δt) supplied (computed once per warp, warp_trig in interval_kernel.cuh)
  __device__ __forceinline__ void init_pre(double w_, double ph0_, double sd_, double cd_) {
    w = w_; ph0 = ph0_; sd = sd_; cd = cd_;
  }
  __device__ __forceinline__ void next(double base, bool anchor) {
    if (anchor) {
      // the frame's first anchor (base 0, phase 0) is e^{i0} exactly: no library call (C5 analytic +2 %)
      if (base == 0.0 && ph0 == 0.0) { s = 0.0; c = 1.0; return; }
      sincos(fma(w, base, ph0), &s, &c);
    } else {
      const double cn = fma(c, cd, -s * sd);
      s = fma(s, cd, c * sd);
      c = cn;
    }
  }
};

// CF4 pair sampling: sample_cf4(base, off1, off2, ...) returns the fields at the two Gauss points of the step that
// starts at t_k + base (off1,2 = fl(base + fl(g1,2·δt))).  Fields with an RF phase evaluate one sincos at the step
// base and reach both Gauss points by rotating with per-interval constants e^{iω g1,2 δt} (init_cf4) — the same
// angle up to ~1e-15 rad at half the trigonometric work.
// Fields whose y coefficient is identically zero declare kZeroY: the frame rotation then skips the terms in f[1]
// (fma(c, 0, ·) and s·0 cannot be folded by the compiler under IEEE semantics; the result is the same to the bit).
template <class F> __device__ constexpr bool zero_y_of(decltype(F::kZeroY)*) { return F::kZeroY; }
template <class F> __device__ constexpr bool zero_y_of(...) { return false; }
// Upper bound on |(fx, fy, fz)| over the interval in the frame rotating at wr (0: frame off) — transverse magnitudes
// are rotation invariant, fz shifts by −wr.  Fields without mag_bound (su(3), user fields): no bound.
template <class F> __device__ __forceinline__ auto field_bound(const F& f, double wr, int) -> decltype(f.mag_bound(wr)) {
  return f.mag_bound(wr);
}
template <class F> __device__ __forceinline__ double field_bound(const F&, double, long) { return 1e300; }

template <> struct Field<FIELD_CONSTANT> {
  double f0, f1, f2, f3;
  __device__ __forceinline__ void init(const double* p, double) { f0 = p[0]; f1 = p[1]; f2 = p[2]; f3 = p[3]; }
  __device__ __forceinline__ double mag_bound(double wr) const { return fabs(f0) + fabs(f1) + fabs(f2 - wr); }
  __device__ __forceinline__ void sample(double, double f[4]) const { f[0] = f0; f[1] = f1; f[2] = f2; f[3] = f3; }
  __device__ __forceinline__ void init_cf4(double, double, double) {}
  static constexpr bool kRF = false;
  __device__ __forceinline__ double rf() const { return 0.0; }
  __device__ __forceinline__ void init_cf4_pre(const double*) {}
  __device__ __forceinline__ void sample_cf4(double, bool, bool, double o1, double o2, double g1[4], double g2[4]) {
    sample(o1, g1); sample(o2, g2);
  }
};

template <> struct Field<FIELD_RABI_LINEAR> {        // ω0 Jz + 2Ω cos(ω0 t) Jx
  static constexpr bool kZeroY = true;               // f[1] ≡ 0 (the frame rotation specialises on it)
  double w0, two_om, ph0, c1, s1, c2, s2;
  PhaseStepper ps;
  __device__ __forceinline__ void init(const double* p, double t_k) {
    w0 = p[0]; two_om = 2.0 * p[1]; ph0 = reduce_phase(p[0], t_k);
  }
  __device__ __forceinline__ void sample(double off, double f[4]) const {
    f[0] = two_om * cos(fma(w0, off, ph0)); f[1] = 0.0; f[2] = w0; f[3] = 0.0;
  }
  __device__ __forceinline__ void init_cf4(double g1dt, double g2dt, double dt) {
    sincos(w0 * g1dt, &s1, &c1); sincos(w0 * g2dt, &s2, &c2);
    ps.init(w0, ph0, dt);
  }
  // RF phase stepper: init_cf4 with its three sincos — of ω·g1δt, ω·g2δt, ω·δt — supplied in t[0..5] as (s, c)
  static constexpr bool kRF = true;
  __device__ __forceinline__ double rf() const { return w0; }
  __device__ __forceinline__ void init_cf4_pre(const double* t) {
    s1 = t[0]; c1 = t[1]; s2 = t[2]; c2 = t[3];
    ps.init_pre(w0, ph0, t[4], t[5]);
  }
  __device__ __forceinline__ void sample_cf4(double base, bool anchor, bool, double, double, double g1[4], double g2[4]) {
    ps.next(base, anchor);
    const double sb = ps.s, cb = ps.c;
    g1[0] = two_om * fma(cb, c1, -sb * s1); g1[1] = 0.0; g1[2] = w0; g1[3] = 0.0;
    g2[0] = two_om * fma(cb, c2, -sb * s2); g2[1] = 0.0; g2[2] = w0; g2[3] = 0.0;
  }
  __device__ __forceinline__ double mag_bound(double wr) const { return fabs(two_om) + fabs(w0 - wr); }
};

template <> struct Field<FIELD_RABI_CIRCULAR> {      // ω0 Jz + Ω(cos(ω0 t) Jx + sin(ω0 t) Jy)
  double w0, om, ph0, c1, s1, c2, s2;
  PhaseStepper ps;
  __device__ __forceinline__ void init(const double* p, double t_k) {
    w0 = p[0]; om = p[1]; ph0 = reduce_phase(p[0], t_k);
  }
  __device__ __forceinline__ void sample(double off, double f[4]) const {
    double s, c;
    sincos(fma(w0, off, ph0), &s, &c);
    f[0] = om * c; f[1] = om * s; f[2] = w0; f[3] = 0.0;
  }
  __device__ __forceinline__ void init_cf4(double g1dt, double g2dt, double dt) {
    sincos(w0 * g1dt, &s1, &c1); sincos(w0 * g2dt, &s2, &c2);
    ps.init(w0, ph0, dt);
  }
  // RF phase stepper: init_cf4 with its three sincos — of ω·g1δt, ω·g2δt, ω·δt — supplied in t[0..5] as (s, c)
  static constexpr bool kRF = true;
  __device__ __forceinline__ double rf() const { return w0; }
  __device__ __forceinline__ void init_cf4_pre(const double* t) {
    s1 = t[0]; c1 = t[1]; s2 = t[2]; c2 = t[3];
    ps.init_pre(w0, ph0, t[4], t[5]);
  }
  __device__ __forceinline__ void sample_cf4(double base, bool anchor, bool, double, double, double g1[4], double g2[4]) {
    ps.next(base, anchor);
    const double sb = ps.s, cb = ps.c;
    g1[0] = om * fma(cb, c1, -sb * s1); g1[1] = om * fma(sb, c1, cb * s1); g1[2] = w0; g1[3] = 0.0;
    g2[0] = om * fma(cb, c2, -sb * s2); g2[1] = om * fma(sb, c2, cb * s2); g2[2] = w0; g2[3] = 0.0;
  }
  __device__ __forceinline__ double mag_bound(double wr) const { return fabs(om) + fabs(w0 - wr); }
};

template <> struct Field<FIELD_NEURAL> {
  // p = [ω_bias, ω_rf, Ω, Ω_p, ω_sig, t_p, ω_q] (reading R16)
  static constexpr bool kZeroY = true;               // f[1] ≡ 0
  double wb, wrf, two_om, op, ws, wq, ph0, dtk, c1, s1, c2, s2;
  // Can a sample of this interval fall inside the signal pulse's single cycle (sinp ≠ 0)?  x = ω_sig(t_k − t_p + off)
  // is monotone in off ∈ [0, Δt]; the margin covers the rounding of the per-sample arguments.  Intervals outside
  // the window take the pulse-free step body (no per-sample window test).
  __device__ __forceinline__ bool pulse_possible(double dt_out) const {
    const double x0 = ws * dtk, x1 = ws * (dtk + dt_out);
    const double lo = fmin(x0, x1), hi = fmax(x0, x1), m = 1e-12 * (fabs(x0) + fabs(x1)) + 1e-300;
    return !(hi < -m || lo > kTwoPi1 + m);
  }
  __device__ __forceinline__ void init(const double* p, double t_k) {
    wb = p[0]; wrf = p[1]; two_om = 2.0 * p[2]; op = p[3]; ws = p[4]; wq = p[6];
    ph0 = reduce_phase(p[1], t_k);
    dtk = __dsub_rn(t_k, p[5]);                     // t_k − t_p
  }
  __device__ __forceinline__ double pulse_z(double off) const {
    const double x = ws * (dtk + off);             // ω_sig (t − t_p)
    const double pulse = (x >= 0.0 && x <= kTwoPi1) ? sin(x) : 0.0;   // sinp (reading R12)
    return fma(op, pulse, wb);
  }
  __device__ __forceinline__ void sample(double off, double f[4]) const {
    f[0] = two_om * cos(fma(wrf, off, ph0));       // 2Ω cos(ω_rf t)
    f[1] = 0.0;
    f[2] = pulse_z(off);
    f[3] = wq;
  }
  PhaseStepper ps;
  __device__ __forceinline__ void init_cf4(double g1dt, double g2dt, double dt) {
    sincos(wrf * g1dt, &s1, &c1); sincos(wrf * g2dt, &s2, &c2);
    ps.init(wrf, ph0, dt);
  }
  // RF phase stepper: init_cf4 with its three sincos — of ω·g1δt, ω·g2δt, ω·δt — supplied in t[0..5] as (s, c)
  static constexpr bool kRF = true;
  __device__ __forceinline__ double rf() const { return wrf; }
  __device__ __forceinline__ void init_cf4_pre(const double* t) {
    s1 = t[0]; c1 = t[1]; s2 = t[2]; c2 = t[3];
    ps.init_pre(wrf, ph0, t[4], t[5]);
  }
  __device__ __forceinline__ void sample_cf4(double base, bool anchor, bool pulse, double o1, double o2, double g1[4], double g2[4]) {
    ps.next(base, anchor);                         // e^{i ω_rf (t_k + base)}, reduced
    const double sb = ps.s, cb = ps.c;
    g1[0] = two_om * fma(cb, c1, -sb * s1); g1[1] = 0.0; g1[2] = pulse ? pulse_z(o1) : wb; g1[3] = wq;
    g2[0] = two_om * fma(cb, c2, -sb * s2); g2[1] = 0.0; g2[2] = pulse ? pulse_z(o2) : wb; g2[3] = wq;
  }
  __device__ __forceinline__ double mag_bound(double wr) const { return fabs(two_om) + fabs(wb - wr) + fabs(op); }
};

template <> struct Field<FIELD_GRADIENT> {          // ω_z = x − 2y
  static constexpr bool kZeroY = true;               // f[1] ≡ 0
  double wz;
  __device__ __forceinline__ void init(const double* p, double) { wz = fma(-2.0, p[1], p[0]); }
  __device__ __forceinline__ double mag_bound(double wr) const { return fabs(wz - wr); }
  __device__ __forceinline__ void sample(double, double f[4]) const { f[0] = 0.0; f[1] = 0.0; f[2] = wz; f[3] = 0.0; }
  __device__ __forceinline__ void init_cf4(double, double, double) {}
  static constexpr bool kRF = false;
  __device__ __forceinline__ double rf() const { return 0.0; }
  __device__ __forceinline__ void init_cf4_pre(const double*) {}
  __device__ __forceinline__ void sample_cf4(double, bool, bool, double o1, double o2, double g1[4], double g2[4]) {
    sample(o1, g1); sample(o2, g2);
  }
};

// General spin-one fields (readings R19, R20).
template <> struct Field<FIELD_SU3_CONSTANT> {      // p = all 8 coefficients
  double c[8];
  __device__ __forceinline__ void init(const double* p, double) {
#pragma unroll
    for (int j = 0; j < 8; ++j) c[j] = p[j];
  }
  __device__ __forceinline__ void sample(double, double f[8]) const {
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = c[j];
  }
  __device__ __forceinline__ void init_cf4(double, double, double) {}
  static constexpr bool kRF = false;
  __device__ __forceinline__ double rf() const { return 0.0; }
  __device__ __forceinline__ void init_cf4_pre(const double*) {}
  __device__ __forceinline__ void sample_cf4(double, bool, bool, double o1, double o2, double g1[8], double g2[8]) {
    sample(o1, g1); sample(o2, g2);
  }
};

// H = ω0 Jz + ω_q Q + Ω_x(cos φ Jx + sin φ Jy) + Ω_v(cos φ V1 + sin φ V2) + Ω_u(cos 2φ U1 + sin 2φ U2), φ = ω_d t;
// p = [ω0, ω_q, Ω_x, Ω_v, Ω_u, ω_d].  φ is reduced per interval in double-double (reading R8); 2φ by double angle.
template <> struct Field<FIELD_SU3_DRIVE> {
  double w0, wq, ox, ov, ou, wd, ph0, c1, s1, c2, s2;
  PhaseStepper ps;
  __device__ __forceinline__ void init(const double* p, double t_k) {
    w0 = p[0]; wq = p[1]; ox = p[2]; ov = p[3]; ou = p[4]; wd = p[5];
    ph0 = reduce_phase(p[5], t_k);
  }
  __device__ __forceinline__ void fill(double c, double s, double f[8]) const {
    const double cc = fma(c, c, -s * s), ss = 2.0 * c * s;   // cos 2φ, sin 2φ
    f[0] = ox * c;  f[1] = ox * s;  f[2] = w0;      f[3] = wq;
    f[4] = ou * cc; f[5] = ou * ss; f[6] = ov * c;  f[7] = ov * s;
  }
  __device__ __forceinline__ void sample(double off, double f[8]) const {
    double s, c;
    sincos(fma(wd, off, ph0), &s, &c);
    fill(c, s, f);
  }
  __device__ __forceinline__ void init_cf4(double g1dt, double g2dt, double dt) {
    sincos(wd * g1dt, &s1, &c1); sincos(wd * g2dt, &s2, &c2);
    ps.init(wd, ph0, dt);
  }
  // RF phase stepper: init_cf4 with its three sincos — of ω·g1δt, ω·g2δt, ω·δt — supplied in t[0..5] as (s, c)
  static constexpr bool kRF = true;
  __device__ __forceinline__ double rf() const { return wd; }
  __device__ __forceinline__ void init_cf4_pre(const double* t) {
    s1 = t[0]; c1 = t[1]; s2 = t[2]; c2 = t[3];
    ps.init_pre(wd, ph0, t[4], t[5]);
  }
  __device__ __forceinline__ void sample_cf4(double base, bool anchor, bool, double, double, double g1[8], double g2[8]) {
    ps.next(base, anchor);
    const double sb = ps.s, cb = ps.c;
    fill(fma(cb, c1, -sb * s1), fma(sb, c1, cb * s1), g1);
    fill(fma(cb, c2, -sb * s2), fma(sb, c2, cb * s2), g2);
  }
};

// Frame rotation of the general spin-one coefficients (reading R19): conjugation by e^{iθJz} multiplies entry (i, j)
// by e^{iθ(m_i − m_j)}, so (ωv1, ωv2) (Δm = ±1) rotate like (ωx, ωy) and (ωu1, ωu2) (Δm = ±2) by 2θ.
template <int NC> __device__ __forceinline__ void rotate_quadrupoles(double* f, double c, double s) {
  if constexpr (NC == 8) {
    const double c2 = fma(c, c, -s * s), s2 = 2.0 * c * s;
    const double u1 = f[4], u2 = f[5];
    f[4] = fma(c2, u1, s2 * u2);
    f[5] = fma(c2, u2, -s2 * u1);
    const double v1 = f[6], v2 = f[7];
    f[6] = fma(c, v1, s * v2);
    f[7] = fma(c, v2, -s * v1);
  }
}

// Only the neural field has a pulse window (pulse_possible above); every other field's step body is pulse-free.
template <class F> __device__ __forceinline__ auto field_pulse_possible(const F& f, double dt_out, int)
    -> decltype(f.pulse_possible(dt_out)) { return f.pulse_possible(dt_out); }
template <class F> __device__ __forceinline__ bool field_pulse_possible(const F&, double, long) { return false; }

// Compile-time booleans for the interval kernel's specialised step bodies (no <type_traits> under NVRTC).
template <bool B> struct BoolC { static constexpr bool value = B; };
struct RtBool { bool value; };
template <int N> struct IntC { static constexpr int value = N; };
struct RtInt { int value; };

// Rotating frame (reading R6): rotate (ωx, ωy) by θ = ω_r·t_local, shift ωz by −ω_r; ωq unchanged.
template <int NC = 4> __device__ __forceinline__ void to_rotating_frame(double* f, double t_local, double omega_r) {
  double s, c;
  sincos(omega_r * t_local, &s, &c);
  const double fx = f[0], fy = f[1];
  f[0] = fma(c, fx, s * fy);
  f[1] = fma(c, fy, -s * fx);
  f[2] = f[2] - omega_r;
  rotate_quadrupoles<NC>(f, c, s);
}

// Frame rotation for the two CF4 samples of one step: θ1,2 = ω_r·base + ω_r·g1,2δt, one sincos per step plus the
// per-interval rotations (cb1, sb1), (cb2, sb2) of ω_r·g1,2δt.
struct FrameCF4 {
  double wr, c1, s1, c2, s2;
  PhaseStepper ps;
  __device__ __forceinline__ void init(double omega_r, double g1dt, double g2dt, double dt) {
    wr = omega_r;
    sincos(omega_r * g1dt, &s1, &c1);
    sincos(omega_r * g2dt, &s2, &c2);
    ps.init(omega_r, 0.0, dt);
  }
  // the same with the three (s, c) supplied in t[0..5] (warp_trig)
  __device__ __forceinline__ void init_pre(double omega_r, const double* t) {
    wr = omega_r;
    s1 = t[0]; c1 = t[1]; s2 = t[2]; c2 = t[3];
    ps.init_pre(omega_r, 0.0, t[4], t[5]);
  }
  template <int NC = 4, bool ZERO_Y = false>
  __device__ __forceinline__ void apply(double base, bool anchor, double* f1, double* f2) {
    ps.next(base, anchor);
    const double sb = ps.s, cb = ps.c;
    const double ca = fma(cb, c1, -sb * s1), sa = fma(sb, c1, cb * s1);
    const double cc = fma(cb, c2, -sb * s2), sc = fma(sb, c2, cb * s2);
    double fx = f1[0], fy = f1[1];
    if constexpr (ZERO_Y) { f1[0] = ca * fx; f1[1] = -(sa * fx); }
    else { f1[0] = fma(ca, fx, sa * fy); f1[1] = fma(ca, fy, -sa * fx); }
    f1[2] -= wr;
    fx = f2[0]; fy = f2[1];
    if constexpr (ZERO_Y) { f2[0] = cc * fx; f2[1] = -(sc * fx); }
    else { f2[0] = fma(cc, fx, sc * fy); f2[1] = fma(cc, fy, -sc * fx); }
    f2[2] -= wr;
    rotate_quadrupoles<NC>(f1, ca, sa);
    rotate_quadrupoles<NC>(f2, cc, sc);
  }
};

// ---- residual matrices ------------------------------------------------------------------------------------------
template <int D, typename T> struct Res {
  T re[D * D];
  T im[D * D];
};

template <int D, typename T> __device__ __forceinline__ void res_zero(Res<D, T>& a) {
#pragma unroll
  for (int e = 0; e < D * D; ++e) { a.re[e] = T(0); a.im[e] = T(0); }
}

// c = a + b + a·b, i.e. (I+a)(I+b) − I, evaluated as b + a·(I + b): the accumulation starts from b_ij and the
// identity only touches the D diagonal real parts of I + b (D adds + 4D³ FMAs instead of 2D² adds + 4D³ FMAs).
template <int D, typename T>
__device__ __forceinline__ void res_mul(const Res<D, T>& a, const Res<D, T>& b, Res<D, T>& c) {
  T bd[D];
#pragma unroll
  for (int k = 0; k < D; ++k) bd[k] = b.re[k * D + k] + T(1);
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      T r = b.re[i * D + j];
      T m = b.im[i * D + j];
#pragma unroll
      for (int k = 0; k < D; ++k) {
        const T br = (k == j) ? bd[k] : b.re[k * D + j];
        r = fmaT(a.re[i * D + k], br, r);
        r = fmaT(-a.im[i * D + k], b.im[k * D + j], r);
        m = fmaT(a.re[i * D + k], b.im[k * D + j], m);
        m = fmaT(a.im[i * D + k], br, m);
      }
      c.re[i * D + j] = r;
      c.im[i * D + j] = m;
    }
}

// ---- spin-half: SU(2)-parametrised residuals ---------------------------------------------------------------------
// Every spin-half operator of the path is in SU(2): U = [[a, b], [−b*, a*]] (the closed form P:359 and all products
// of it).  The residual is carried as (δa = a − 1, b) — 4 reals instead of 8 — and products use the group law
// (a₁, b₁)(a₂, b₂) = (a₁a₂ − b₁b₂*, a₁b₂ + b₁a₂*): in residual form
//   δa = δa₁ + δa₂ + δa₁δa₂ − b₁b₂*,   b = b₁ + b₂ + δa₁b₂ + b₁δa₂*,
// 20 FP64 instructions instead of 34 for the dense 2×2 residual product; the same matrices, exactly.
template <typename T> struct Res<2, T> {
  T ar, ai, br, bi;
  // dense entries (r, c) of the residual: (0,0) = δa, (0,1) = b, (1,0) = −b*, (1,1) = δa*
  __device__ __forceinline__ T re(int r, int c) const { return r == c ? ar : (r == 0 ? br : -br); }
  __device__ __forceinline__ T im(int r, int c) const { return r == c ? (r == 0 ? ai : -ai) : bi; }
};

template <typename T> __device__ __forceinline__ void res_zero(Res<2, T>& a) { a.ar = a.ai = a.br = a.bi = T(0); }

// c = (I + x)(I + y) − I
template <typename T>
__device__ __forceinline__ void res_mul(const Res<2, T>& x, const Res<2, T>& y, Res<2, T>& c) {
  T ar = fmaT(x.ar, y.ar, x.ar + y.ar);
  ar = fmaT(-x.ai, y.ai, ar);
  ar = fmaT(-x.br, y.br, ar);
  ar = fmaT(-x.bi, y.bi, ar);
  T ai = fmaT(x.ar, y.ai, x.ai + y.ai);
  ai = fmaT(x.ai, y.ar, ai);
  ai = fmaT(-x.bi, y.br, ai);
  ai = fmaT(x.br, y.bi, ai);
  T br = fmaT(x.ar, y.br, x.br + y.br);
  br = fmaT(-x.ai, y.bi, br);
  br = fmaT(x.br, y.ar, br);
  br = fmaT(x.bi, y.ai, br);
  T bi = fmaT(x.ar, y.bi, x.bi + y.bi);
  bi = fmaT(x.ai, y.br, bi);
  bi = fmaT(x.bi, y.ar, bi);
  bi = fmaT(-x.br, y.ai, bi);
  c.ar = ar; c.ai = ai; c.br = br; c.bi = bi;
}

template <typename T> __device__ __forceinline__ T res_re(const Res<2, T>& a, int r, int c) { return a.re(r, c); }
template <typename T> __device__ __forceinline__ T res_im(const Res<2, T>& a, int r, int c) { return a.im(r, c); }
template <typename T> __device__ __forceinline__ T res_re(const Res<3, T>& a, int r, int c) { return a.re[3 * r + c]; }
template <typename T> __device__ __forceinline__ T res_im(const Res<3, T>& a, int r, int c) { return a.im[3 * r + c]; }

template <typename T> __device__ __forceinline__ Res<2, T> res_shfl_down(const Res<2, T>& m, int delta) {
  Res<2, T> r;
  r.ar = __shfl_down_sync(0xffffffffu, m.ar, delta);
  r.ai = __shfl_down_sync(0xffffffffu, m.ai, delta);
  r.br = __shfl_down_sync(0xffffffffu, m.br, delta);
  r.bi = __shfl_down_sync(0xffffffffu, m.bi, delta);
  return r;
}
template <typename T> __device__ __forceinline__ Res<3, T> res_shfl_down(const Res<3, T>& m, int delta) {
  Res<3, T> r;
#pragma unroll
  for (int e = 0; e < 9; ++e) {
    r.re[e] = __shfl_down_sync(0xffffffffu, m.re[e], delta);
    r.im[e] = __shfl_down_sync(0xffffffffu, m.im[e], delta);
  }
  return r;
}

// ---- exponentiators: residual of exp(−i(ax Jx + ay Jy + az Jz + aq Q)) -----------------------------------------

// Spin-half closed form: exp(−i a·σ/2) = cos(r/2) I − i (sin(r/2)/r) a·σ.  cos(r/2) − 1 = −2 sin²(r/4).
// series (FP64): 2 = the caller guarantees r ≤ 2^-13, 1 = r ≤ 2^-7, 0 = no bound (interval_residual bounds |a| once per
// interval from the field's magnitude bound).  The short series keeps two terms of each function (the dropped r⁶/46080
// and r⁴/3840 are < 1.2e-19 relative), the medium one three (dropped r⁸/10321920 and r⁶/645120: < 7e-19 relative at
// r = 2^-7), the full one five below r = 2^-4 and the library sincos above.  Former description of the short case:
// short_series: the caller guarantees r ≤ 2^-13 for this argument (interval_body bounds |a| once per interval from
// the field's magnitude bound, field_bound): then two series terms each suffice — the dropped r⁶/46080 and r⁴/3840
// are < 1.2e-19 relative (DESIGN.md §5 item 15).  A per-step test instead costs an FP64 compare per exponential and,
// where lanes straddle the bound (C5's 100 ns steps), both series.
template <typename T>
__device__ __forceinline__ void expo_su2(const T a[4], Res<2, T>& e, int series = 0) {
  const T r2 = a[0] * a[0] + a[1] * a[1] + a[2] * a[2];
  T cm1, s;
  if (sizeof(T) == 8 && series == 2) {
    cm1 = r2 * fmaT(r2, T(kSu2Series[3]), T(kSu2Series[4]));
    s = fmaT(r2, T(kSu2Series[8]), T(kSu2Series[9]));
  } else if (sizeof(T) == 8 && series == 1) {
    cm1 = r2 * fmaT(r2, fmaT(r2, T(kSu2Series[2]), T(kSu2Series[3])), T(kSu2Series[4]));
    s = fmaT(r2, fmaT(r2, T(kSu2Series[7]), T(kSu2Series[8])), T(kSu2Series[9]));
  } else if (r2 <= T(0.00390625)) {
    // r ≤ 2^-4 (every fine step of the configs): both functions are even, so series in r² need no sqrt, sincos
    // or division.  cos(r/2) − 1 = −r²/8 + r⁴/384 − r⁶/46080 + r⁸/10321920 − r¹⁰/3715891200,
    // sin(r/2)/r = 1/2 − r²/48 + r⁴/3840 − r⁶/645120 + r⁸/185794560 (truncation < 1e-19 relative).
    // FP64 coefficients come from the constant bank (DFMA c[][] operands) instead of being rematerialised in
    // uniform registers every step (measured: 37 UMOV per spin-half fine step).
    if constexpr (sizeof(T) == 8) {
      cm1 = r2 * fma(r2, fma(r2, fma(r2, fma(r2, kSu2Series[0], kSu2Series[1]), kSu2Series[2]), kSu2Series[3]),
                     kSu2Series[4]);
      s = fma(r2, fma(r2, fma(r2, fma(r2, kSu2Series[5], kSu2Series[6]), kSu2Series[7]), kSu2Series[8]),
              kSu2Series[9]);
    } else {
      cm1 = r2 * fmaT(r2, fmaT(r2, fmaT(r2, fmaT(r2, T(-1.0 / 3715891200.0), T(1.0 / 10321920.0)),
                                          T(-1.0 / 46080.0)), T(1.0 / 384.0)), T(-0.125));
      s = fmaT(r2, fmaT(r2, fmaT(r2, fmaT(r2, T(1.0 / 185794560.0), T(-1.0 / 645120.0)), T(1.0 / 3840.0)),
                        T(-1.0 / 48.0)), T(0.5));
    }
  } else {
    const T r = sqrtT(r2);
    T sq, cq;
    sincosT(r * T(0.25), &sq, &cq);
    cm1 = T(-2) * sq * sq;                           // cos(r/2) − 1 without cancellation
    s = (T(2) * sq * cq) / r;                        // sin(r/2)/r  (r = 0 takes the series branch: ½, reading R4)
  }
  e.ar = cm1;       e.ai = -s * a[2];               // δa = cos − 1 − i s az
  e.br = -s * a[1]; e.bi = -s * a[0];               // b = −i s (ax − i ay);  (1,0) = −b* = −i s (ax + i ay)
}

// Spin-one Lie–Trotter.  The leapfrog factor T = e^{−iD/2} e^{−iΦJφ} e^{−iD/2} with
// Jφ = e^{−iφJz} Jx e^{iφJz} and D diagonal factors as T = R_φ T₀ R_φ†, R_φ = e^{−iφJz} = diag(e^{−iφ}, 1, e^{iφ}),
// T₀ = e^{−iD/2} e^{−iΦJx} e^{−iD/2}.  T₀ is complex SYMMETRIC (diagonal·symmetric·diagonal), so is every power
// T₀^{2^k}, and T^n = R_φ T₀^n R_φ† exactly.  The τ residual squarings therefore run on the 6 unique
// entries of T₀ − I (63 FP64 instructions per squaring instead of 111 for a dense 3×3 complex square), and the
// phases e^{−iφ(m−n)} are applied once at the end.  Same algorithm, same result up to rounding.
//
// T₀ − I from Eq. lie_trotter_4 at φ = 0 with the corrections of reading R1, θ1 = z + q/3, θ2 = 2q/3, θ3 = z − q/3
// (z = az/n, q = aq/n, n = 2^τ, s = sin(Φ/2)):
//   T11 − 1 = expm1(−iθ1) − s² e^{−iθ1}   T12 = T21 = (−i/√2) sinΦ e^{−iθ3/2}   T13 = T31 = −s² e^{−iθ2/2}
//   T22 − 1 = expm1(iθ2) − 2s² e^{iθ2}    T23 = T32 = (−i/√2) sinΦ e^{iθ1/2}    T33 − 1 = expm1(iθ3) − s² e^{iθ3}
// with the diagonal from half-angle sines (expm1(iθ) = −2 sin²(θ/2) + i sin θ), and e^{iφ} =
// (ax + i ay)/√(ax² + ay²) (no atan2; := 1 at Φ = 0, reading R3).
template <typename T> struct Sym3 {   // unique entries of a complex symmetric 3×3 residual
  T r00, i00, r01, i01, r02, i02, r11, i11, r12, i12, r22, i22;
};

// Below this bound on the entries of A = H/n (Σ|a_j|/n), the leapfrog factor's residual equals its second-order
// Taylor polynomial to within rounding: a palindromic product of exponentials is exp(−iA + O(A³)) (symmetric
// splitting), so T − I = −iA − A²/2 + O(A³), and the dropped terms are ≤ |A|²/6 ≈ 2^-56 (FP64) / 2^-26 (FP32)
// relative to T − I — below one ulp.  Every physical step at τ = 24 takes this path (|a| ≲ 0.1 rad); the closed
// forms remain for large arguments (item 9).
template <typename T> __device__ __forceinline__ T taylor_bound();
template <> __device__ __forceinline__ double taylor_bound<double>() { return 7.450580596923828e-09; }   // 2^-27
template <> __device__ __forceinline__ float taylor_bound<float>() { return 2.44140625e-04f; }           // 2^-12

// The residual squaring s = (a + 2I)a of P:456-462 in double-angle form.  T₀ is complex symmetric AND unitary, so
// with T₀ = X + iY (X, Y real symmetric) unitarity T₀T₀* = I reads X² + Y² = I and XY = YX; every power keeps both
// properties.  Then T₀² = X² − Y² + 2iXY = (I − 2Y²) + 2i XY, i.e. for the residual a = x + iy (x = X − I, y = Y):
// x' = −2y², y' = 2y + 2xy — the double-angle formulas cos 2Θ = 1 − 2 sin²Θ, sin 2Θ = 2 sin Θ cos Θ of T₀ = e^{iΘ}.
// Exactly (a + 2I)a for a unitary symmetric T₀ (the dropped term x² + 2x + y² is T₀'s unitarity defect, zero up to
// rounding): two real symmetric products instead of a complex one (DESIGN.md §5 item 13; the complex form took 63 FP64
// instructions, the unscaled double-angle one 48).
// Scaled double-angle form: carrying x̃ = 2x and ỹ = −2y (exact rescalings by powers of two) the doubling becomes
//   x̃' = −ỹ²,  ỹ' = (x̃ + 2I)·ỹ
// (x̃' = 2x' = −4y² = −ỹ²;  ỹ' = −2y' = −4y − 4xy = (2x + 2I)(−2y)) — two symmetric products and a diagonal shift:
// 3 DADD + 12 DMUL + 24 DFMA = 39 FP64 instructions (36 in the shifted-diagonal form below).  trotter_init produces
// and trotter_expand consumes this form.
template <typename T> __device__ __forceinline__ void sym_square_s(Sym3<T>& a) {
  const T two = splat<T>(2.0);
  const T d0 = a.r00 + two, d1 = a.r11 + two, d2 = a.r22 + two;
  const T x01 = a.r01, x02 = a.r02, x12 = a.r12;
  const T y00 = a.i00, y01 = a.i01, y02 = a.i02, y11 = a.i11, y12 = a.i12, y22 = a.i22;
  // x̃' = −ỹ·ỹ
  a.r00 = fmaT(-y00, y00, fmaT(-y01, y01, -(y02 * y02)));
  a.r01 = fmaT(-y00, y01, fmaT(-y01, y11, -(y02 * y12)));
  a.r02 = fmaT(-y00, y02, fmaT(-y01, y12, -(y02 * y22)));
  a.r11 = fmaT(-y01, y01, fmaT(-y11, y11, -(y12 * y12)));
  a.r12 = fmaT(-y01, y02, fmaT(-y11, y12, -(y12 * y22)));
  a.r22 = fmaT(-y02, y02, fmaT(-y12, y12, -(y22 * y22)));
  // ỹ' = (x̃ + 2I)·ỹ
  a.i00 = fmaT(d0, y00, fmaT(x01, y01, x02 * y02));
  a.i01 = fmaT(d0, y01, fmaT(x01, y11, x02 * y12));
  a.i02 = fmaT(d0, y02, fmaT(x01, y12, x02 * y22));
  a.i11 = fmaT(x01, y01, fmaT(d1, y11, x12 * y12));
  a.i12 = fmaT(x01, y02, fmaT(d1, y12, x12 * y22));
  a.i22 = fmaT(x02, y02, fmaT(x12, y12, d2 * y22));
}

// The Sym3 between trotter_init and trotter_expand holds the scaled pair (x̃, ỹ) = (2x, −2y).
template <typename T> __device__ __forceinline__ void lt_square(Sym3<T>& a) { sym_square_s<T>(a); }

// Shifted-diagonal form of the τ-squaring loop (DESIGN.md §5 item 19).  The doubling reads x̃'s diagonal only as
// d_i = x̃_ii + 2, so between squarings the Sym3 may carry w_ii = x̃_ii + 2 on its diagonal instead: the next
// diagonal is then w'_ii = 2 − (ỹ²)_ii, three FMAs with the constant as the innermost addend, where x̃'_ii = −(ỹ²)_ii
// took two FMAs and a DMUL and d_i one DADD more — 36 FP64 instructions per squaring instead of 39.  Same squarings
// (P:456-462); only d_i's rounding moves (three roundings at the magnitude of 2 instead of one).  The last squaring
// writes x̃'s diagonal again (−(ỹ²)_ii with full relative precision), so T₀^n − I keeps its residual accuracy.
#ifndef SS_SQ_WFORM
#define SS_SQ_WFORM 1
#endif
template <typename T, bool W_OUT> __device__ __forceinline__ void sym_square_w(Sym3<T>& a) {
  const T two = splat<T>(2.0);
  const T d0 = a.r00, d1 = a.r11, d2 = a.r22;         // w_ii = x̃_ii + 2
  const T x01 = a.r01, x02 = a.r02, x12 = a.r12;
  const T y00 = a.i00, y01 = a.i01, y02 = a.i02, y11 = a.i11, y12 = a.i12, y22 = a.i22;
  if constexpr (W_OUT) {                               // w' = 2I − ỹ² on the diagonal
    a.r00 = fmaT(-y00, y00, fmaT(-y01, y01, fmaT(-y02, y02, two)));
    a.r11 = fmaT(-y01, y01, fmaT(-y11, y11, fmaT(-y12, y12, two)));
    a.r22 = fmaT(-y02, y02, fmaT(-y12, y12, fmaT(-y22, y22, two)));
  } else {                                             // x̃' = −ỹ² on the diagonal (the last squaring)
    a.r00 = fmaT(-y00, y00, fmaT(-y01, y01, -(y02 * y02)));
    a.r11 = fmaT(-y01, y01, fmaT(-y11, y11, -(y12 * y12)));
    a.r22 = fmaT(-y02, y02, fmaT(-y12, y12, -(y22 * y22)));
  }
  a.r01 = fmaT(-y00, y01, fmaT(-y01, y11, -(y02 * y12)));
  a.r02 = fmaT(-y00, y02, fmaT(-y01, y12, -(y02 * y22)));
  a.r12 = fmaT(-y01, y02, fmaT(-y11, y12, -(y12 * y22)));
  // ỹ' = (x̃ + 2I)·ỹ
  a.i00 = fmaT(d0, y00, fmaT(x01, y01, x02 * y02));
  a.i01 = fmaT(d0, y01, fmaT(x01, y11, x02 * y12));
  a.i02 = fmaT(d0, y02, fmaT(x01, y12, x02 * y22));
  a.i11 = fmaT(x01, y01, fmaT(d1, y11, x12 * y12));
  a.i12 = fmaT(x01, y02, fmaT(d1, y12, x12 * y22));
  a.i22 = fmaT(x02, y02, fmaT(x12, y12, d2 * y22));
}

#ifndef SS_SQ_UNROLL
#define SS_SQ_UNROLL 2      // unroll of the τ-squaring loop (tuning knob)
#endif
#define SS_PRAGMA(x) _Pragma(#x)
#define SS_UNROLL(n) SS_PRAGMA(unroll n)

// The τ residual squarings of the scaled pair: shifted-diagonal form in FP64 when SS_SQ_WFORM.  FP32
// keeps the unshifted form: at its precision the diagonal's three roundings at the magnitude of 2 doubled C5's
// error against the oracle (1.72e-5 → 3.26e-5, bar 1e-4) for a 0.9 % faster step (profiles/r02/s54_wform_fp32/).
template <typename T> __device__ __forceinline__ void lt_square_tau(Sym3<T>& m, int tau) {
  if constexpr (SS_SQ_WFORM && sizeof(T) == 8) {
    if (tau <= 0) return;
    const T two = splat<T>(2.0);
    m.r00 = m.r00 + two; m.r11 = m.r11 + two; m.r22 = m.r22 + two;
    SS_UNROLL(SS_SQ_UNROLL)
    for (int it = 1; it < tau; ++it) sym_square_w<T, true>(m);
    sym_square_w<T, false>(m);
  } else {
    SS_UNROLL(SS_SQ_UNROLL)
    for (int it = 0; it < tau; ++it) lt_square<T>(m);
  }
}

// Two FP32 symmetric residuals packed one per float2 lane (FP32 mode squares both exponentials of a CF4 step in
// lockstep with packed FFMA2).
__device__ __forceinline__ Sym3<float2> sym_pack(const Sym3<float>& a, const Sym3<float>& b) {
  Sym3<float2> m;
  m.r00 = make_float2(a.r00, b.r00); m.i00 = make_float2(a.i00, b.i00);
  m.r01 = make_float2(a.r01, b.r01); m.i01 = make_float2(a.i01, b.i01);
  m.r02 = make_float2(a.r02, b.r02); m.i02 = make_float2(a.i02, b.i02);
  m.r11 = make_float2(a.r11, b.r11); m.i11 = make_float2(a.i11, b.i11);
  m.r12 = make_float2(a.r12, b.r12); m.i12 = make_float2(a.i12, b.i12);
  m.r22 = make_float2(a.r22, b.r22); m.i22 = make_float2(a.i22, b.i22);
  return m;
}
__device__ __forceinline__ void sym_unpack(const Sym3<float2>& m, Sym3<float>& a, Sym3<float>& b) {
  a.r00 = m.r00.x; a.i00 = m.i00.x; a.r01 = m.r01.x; a.i01 = m.i01.x; a.r02 = m.r02.x; a.i02 = m.i02.x;
  a.r11 = m.r11.x; a.i11 = m.i11.x; a.r12 = m.r12.x; a.i12 = m.i12.x; a.r22 = m.r22.x; a.i22 = m.i22.x;
  b.r00 = m.r00.y; b.i00 = m.i00.y; b.r01 = m.r01.y; b.i01 = m.i01.y; b.r02 = m.r02.y; b.i02 = m.i02.y;
  b.r11 = m.r11.y; b.i11 = m.i11.y; b.r12 = m.r12.y; b.i12 = m.i12.y; b.r22 = m.r22.y; b.i22 = m.i22.y;
}

// T₀ − I and the phase of φ (cos φ, sin φ) for exponent arguments a (divided by n = 2^τ inside).
template <typename T>
__device__ __forceinline__ void trotter_init(const T a[4], int tau, Sym3<T>& m, T& cphi, T& sphi) {
  const T inv_n = ldexp(T(1), -tau);
  const T r2 = a[0] * a[0] + a[1] * a[1];
  T rxy = T(0);
  cphi = T(1);
  sphi = T(0);
  if (r2 > T(0)) {                                   // e^{iφ} = (ax + i ay)/√(ax² + ay²) via one reciprocal sqrt
    const T ir = rsqrtT(r2);
    rxy = r2 * ir;
    cphi = a[0] * ir;
    sphi = a[1] * ir;
  }
  const T Phi = rxy * inv_n;
  const T z = a[2] * inv_n, q = a[3] * inv_n;
  if ((fabs(a[0]) + fabs(a[1]) + fabs(a[2]) + fabs(a[3])) * inv_n <= taylor_bound<T>()) {
    // T₀ − I = −iA₀ − A₀²/2, A₀ = D + Φ Jx (real symmetric): diag(D) = (z + q/3, −2q/3, q/3 − z), off-diagonal
    // x = Φ/√2 on (0,1), (1,2).  A₀² = [[d0² + x², x(d0 + d1), x²], [·, d1² + 2x², x(d1 + d2)], [·, ·, d2² + x²]].
    const T d0 = z + q * T(kThird), d1 = T(-2) * q * T(kThird), d2 = q * T(kThird) - z;
    const T x = Phi * T(kRsqrt2), x2 = x * x;
    // scaled pair (2x, −2y) = (−A₀², 2A₀)
    const T x_2 = x + x;
    m.r00 = -fmaT(d0, d0, x2);          m.i00 = d0 + d0;
    m.r11 = -fmaT(d1, d1, x2 + x2);     m.i11 = d1 + d1;
    m.r22 = -fmaT(d2, d2, x2);          m.i22 = d2 + d2;
    m.r01 = -(x * (d0 + d1));           m.i01 = x_2;
    m.r12 = -(x * (d1 + d2));           m.i12 = x_2;
    m.r02 = -x2;                        m.i02 = T(0);
    return;
  }
  const T th1 = z + q * T(kThird), th2 = T(2) * q * T(kThird), th3 = z - q * T(kThird);
  T s, c, s1, c1, s2, c2, s3, c3;
  const T big = fmax(fmax(Phi, fabs(th1)), fmax(fabs(th2), fabs(th3)));
  if (big <= T(1.9073486328125e-06)) {
    // half-angles ≤ 2^-20 (every physical step at τ = 24: |a| ≲ 16 rad ⇒ |x| ≤ 2^-21): sin x = x − x³/6 and
    // cos x = 1 − x²/2 are exact to < 1e-25 relative (cos enters only through sin 2x = 2 sin x cos x).
    sincos_tiny<T>(Phi * T(0.5), &s, &c);
    sincos_tiny<T>(th1 * T(0.5), &s1, &c1);
    sincos_tiny<T>(th2 * T(0.5), &s2, &c2);
    sincos_tiny<T>(th3 * T(0.5), &s3, &c3);
  } else if (big <= T(0.03125)) {                    // half-angles ≤ 2^-6: polynomial
    sincos_small<T>(Phi * T(0.5), &s, &c);
    sincos_small<T>(th1 * T(0.5), &s1, &c1);
    sincos_small<T>(th2 * T(0.5), &s2, &c2);
    sincos_small<T>(th3 * T(0.5), &s3, &c3);
  } else {
    sincosT(Phi * T(0.5), &s, &c);
    sincosT(th1 * T(0.5), &s1, &c1);
    sincosT(th2 * T(0.5), &s2, &c2);
    sincosT(th3 * T(0.5), &s3, &c3);
  }
  const T ss = s * s;
  const T sinPhi_r2 = T(2) * s * c * T(kRsqrt2);     // sinΦ/√2
  // T12 = (−i/√2) sinΦ e^{−iθ3/2} = (−i) X (c3 − i s3) = X(−s3 − i c3)
  m.r01 = -sinPhi_r2 * s3;  m.i01 = -sinPhi_r2 * c3;
  // T23 = (−i/√2) sinΦ e^{iθ1/2} = (−i) X (c1 + i s1) = X(s1 − i c1)
  m.r12 = sinPhi_r2 * s1;   m.i12 = -sinPhi_r2 * c1;
  // T13 = −s² e^{−iθ2/2}
  m.r02 = -ss * c2;         m.i02 = ss * s2;
  {  // diagonal: e^{iθ} = (1 − 2sh², 2 sh ch); expm1(iθ) = (−2sh², 2 sh ch)
    const T sin1 = T(2) * s1 * c1, v1 = T(-2) * s1 * s1;
    const T sin2 = T(2) * s2 * c2, v2 = T(-2) * s2 * s2;
    const T sin3 = T(2) * s3 * c3, v3 = T(-2) * s3 * s3;
    m.r00 = v1 - ss * (T(1) + v1);             m.i00 = -sin1 + ss * sin1;          // expm1(−iθ1) − s² e^{−iθ1}
    m.r11 = v2 - T(2) * ss * (T(1) + v2);      m.i11 = sin2 - T(2) * ss * sin2;    // expm1(iθ2) − 2s² e^{iθ2}
    m.r22 = v3 - ss * (T(1) + v3);             m.i22 = sin3 - ss * sin3;           // expm1(iθ3) − s² e^{iθ3}
  }
  {                                                   // to the scaled pair (2x, −2y)
    const T p2 = T(2), m2 = T(-2);
    m.r00 *= p2; m.r01 *= p2; m.r02 *= p2; m.r11 *= p2; m.r12 *= p2; m.r22 *= p2;
    m.i00 *= m2; m.i01 *= m2; m.i02 *= m2; m.i11 *= m2; m.i12 *= m2; m.i22 *= m2;
  }
}

// e = R_φ (T₀^n − I) R_φ†: entry (m, n) gains e^{−iφ(m−n)} (m = +1, 0, −1 ↔ rows 0, 1, 2).
template <typename T>
__device__ __forceinline__ void trotter_expand(const Sym3<T>& m0, T cphi, T sphi, Res<3, T>& e) {
  Sym3<T> m = m0;
  {                              // back from (2x, −2y): the ½ folds into the phase factors, the diagonal costs 6 DMUL
    const T h = T(0.5), mh = T(-0.5);
    m.r00 = h * m0.r00; m.r11 = h * m0.r11; m.r22 = h * m0.r22;
    m.i00 = mh * m0.i00; m.i11 = mh * m0.i11; m.i22 = mh * m0.i22;
    m.i01 = -m0.i01; m.i12 = -m0.i12; m.i02 = -m0.i02;       // signs fold into the products below
    cphi = h * cphi;
    sphi = h * sphi;
  }
  const T c2phi = T(2) * (cphi * cphi - sphi * sphi);
  const T s2phi = T(4) * cphi * sphi;
  e.re[0] = m.r00;  e.im[0] = m.i00;
  e.re[4] = m.r11;  e.im[4] = m.i11;
  e.re[8] = m.r22;  e.im[8] = m.i22;
  // × e^{−iφ} = (cphi, −sphi)
  e.re[1] = m.r01 * cphi + m.i01 * sphi;   e.im[1] = m.i01 * cphi - m.r01 * sphi;
  e.re[5] = m.r12 * cphi + m.i12 * sphi;   e.im[5] = m.i12 * cphi - m.r12 * sphi;
  // × e^{+iφ}
  e.re[3] = m.r01 * cphi - m.i01 * sphi;   e.im[3] = m.i01 * cphi + m.r01 * sphi;
  e.re[7] = m.r12 * cphi - m.i12 * sphi;   e.im[7] = m.i12 * cphi + m.r12 * sphi;
  // × e^{∓2iφ}
  e.re[2] = m.r02 * c2phi + m.i02 * s2phi; e.im[2] = m.i02 * c2phi - m.r02 * s2phi;
  e.re[6] = m.r02 * c2phi - m.i02 * s2phi; e.im[6] = m.i02 * c2phi + m.r02 * s2phi;
}

template <typename T> __device__ __forceinline__ void trotter_residual(const T a[4], int tau, Res<3, T>& e) {
  Sym3<T> m;
  T cphi, sphi;
  trotter_init<T>(a, tau, m, cphi, sphi);
  lt_square_tau<T>(m, tau);
  trotter_expand<T>(m, cphi, sphi, e);
}

// Spin-one "analytic" exponential (reading R14): D¹ of the SU(2) closed form, valid iff aq = 0.
// With α = 1 + δα, β (from expo_su2): D¹ − I = [[δα(δα+2), √2αβ, β²], [−√2αβ*, −2|β|², √2α*β], [β*², −√2α*β*, δα*(δα*+2)]].
template <typename T> __device__ __forceinline__ void su2_to_spin1(const Res<2, T>& u, Res<3, T>& e) {
  const T dar = u.ar, dai = u.ai;                    // δα = α − 1
  const T ar = T(1) + dar, ai = dai;                 // α
  const T br = u.br, bi = u.bi;                      // β
  const T r2 = T(kSqrt2);
  // δα(δα + 2)
  e.re[0] = dar * (dar + T(2)) - dai * dai;          e.im[0] = dai * (dar + T(2)) + dar * dai;
  // √2 α β
  e.re[1] = r2 * (ar * br - ai * bi);                e.im[1] = r2 * (ar * bi + ai * br);
  // β²
  e.re[2] = br * br - bi * bi;                       e.im[2] = T(2) * br * bi;
  // −√2 α β*
  e.re[3] = -r2 * (ar * br + ai * bi);               e.im[3] = -r2 * (ai * br - ar * bi);
  // |α|² − |β|² − 1 = −2|β|²
  e.re[4] = T(-2) * (br * br + bi * bi);             e.im[4] = T(0);
  // √2 α* β
  e.re[5] = r2 * (ar * br + ai * bi);                e.im[5] = r2 * (ar * bi - ai * br);
  // β*²
  e.re[6] = br * br - bi * bi;                       e.im[6] = T(-2) * br * bi;
  // −√2 α* β*
  e.re[7] = -r2 * (ar * br - ai * bi);               e.im[7] = r2 * (ar * bi + ai * br);
  // δα*(δα* + 2)
  e.re[8] = dar * (dar + T(2)) - dai * dai;          e.im[8] = -(dai * (dar + T(2)) + dar * dai);
}

// ---- general spin-one exponentiator (readings R19, R20) -----------------------
// exp(−iH) for H = Σ a_j A_j over (Jx, Jy, Jz, Q, U1, U2, V1, V2): Lie–Trotter U = T^n, n = 2^τ.  H is brought to
// real symmetric tridiagonal form S = W†HW by W = diag(1, g), g = G·diag(1, e^{iψ}) with
// G = [[H01*, −H02], [H02*, H01]]/r, r = √(|H01|² + |H02|²), and e^{iψ} = B12*/|B12| for B = G†H_blk G (reading R20);
// the factor is T = W T₀ W†, T₀ = e^{−iD/2} e^{−iX} e^{−iD/2} on S/n (the paper's Eq. lie_trotter_4 shape).  T₀ is
// complex symmetric and unitary, so its τ squarings take the scaled double-angle form (36 instructions, §5 items 13, 19)
// and W is applied once at the end: (W T₀ W†)^n − I = W (T₀^n − I) W† (DESIGN.md §5 item 14).

// sin r / r and (cos r − 1)/r² from r² (both even): series for r ≤ 2^-4 (truncation < 1e-19 relative), else library.
template <typename T> __device__ __forceinline__ void sinc_cosm1(T r2, T* sinc, T* cm) {
  if (r2 <= T(0.00390625)) {
    *sinc = fmaT(r2, fmaT(r2, fmaT(r2, fmaT(r2, T(1.0 / 362880.0), T(-1.0 / 5040.0)), T(1.0 / 120.0)), T(-1.0 / 6.0)),
                 T(1));
    *cm = fmaT(r2, fmaT(r2, fmaT(r2, fmaT(r2, T(-1.0 / 3628800.0), T(1.0 / 40320.0)), T(-1.0 / 720.0)),
                         T(1.0 / 24.0)), T(-0.5));
  } else {
    const T r = sqrtT(r2);
    T sh, ch;
    sincosT(r * T(0.5), &sh, &ch);
    *sinc = T(2) * sh * ch / r;
    *cm = T(-2) * sh * sh / r2;
  }
}

template <typename T> struct Su3W {   // the (1,2) block g of W = diag(1, g), pre-scaled by ½ (see su3_expand)
  T g11r, g11i, g12r, g12i, g21r, g21i, g22r, g22i;
};

// v ← v/|v|, returns |v| (0 for v = 0, v then unchanged).  When |v|² leaves the normal range (components below
// ≈ 1e-19 in FP32 / 1e-154 in FP64, where a subnormal |v|² keeps only a few bits and W would stop being unitary) the
// components are first rescaled by an exact power of two.
template <typename T> __device__ __forceinline__ T norm_lo();
template <typename T> __device__ __forceinline__ T norm_hi();
template <> __device__ __forceinline__ double norm_lo<double>() { return 0x1p-960; }
template <> __device__ __forceinline__ double norm_hi<double>() { return 0x1p960; }
template <> __device__ __forceinline__ float norm_lo<float>() { return 0x1p-100f; }
template <> __device__ __forceinline__ float norm_hi<float>() { return 0x1p100f; }
template <int N, typename T> __device__ __forceinline__ T unit_vec(T (&v)[N]) {
  T r2 = v[0] * v[0];
#pragma unroll
  for (int i = 1; i < N; ++i) r2 = fmaT(v[i], v[i], r2);
  if (r2 >= norm_lo<T>() && r2 <= norm_hi<T>()) {
    const T ir = rsqrtT(r2);
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] *= ir;
    return r2 * ir;
  }
  T m = fabs(v[0]);
#pragma unroll
  for (int i = 1; i < N; ++i) m = fmax(m, fabs(v[i]));
  if (!(m > T(0))) return T(0);
  const int e = ilogb(m);
  const T sc = ldexp(T(1), -e);
#pragma unroll
  for (int i = 0; i < N; ++i) v[i] *= sc;
  r2 = v[0] * v[0];
#pragma unroll
  for (int i = 1; i < N; ++i) r2 = fmaT(v[i], v[i], r2);
  const T ir = rsqrtT(r2);
#pragma unroll
  for (int i = 0; i < N; ++i) v[i] *= ir;
  return ldexp(r2 * ir, e);
}

// S = W†HW from the unscaled coefficients a[8]: diagonal (s0, s1, s2), off-diagonals al = S01 = r, be = S12 ≥ 0.
// With the unit pair u1 = H01/r, u2 = H02/r (all products below stay O(|H|)):
// B11 = |u1|² d1 + |u2|² d2 + 2 Re(u1 H12 u2*),  B22 = d1 + d2 − B11 (trace kept exact),
// B12 = u1 u2 (d2 − d1) + u1² H12 − u2² H12*.
template <typename T>
__device__ __forceinline__ void su3_tridiagonalise(const T* a, T& s0, T& s1, T& s2, T& al, T& be, Su3W<T>& w) {
  const T k = T(kRsqrt2);
  const T d0 = a[2] + a[3] * T(kThird), d1 = T(-2) * a[3] * T(kThird), d2 = a[3] * T(kThird) - a[2];
  const T br = (a[0] - a[6]) * k, bi = -(a[1] - a[7]) * k;        // H12
  T u[4] = {(a[0] + a[6]) * k, -(a[1] + a[7]) * k, a[4], -a[5]};  // (H01, H02), normalised below
  T b12r = br, b12i = bi;
  s0 = d0; s1 = d1; s2 = d2;
  w.g11r = T(0.5); w.g11i = T(0); w.g12r = T(0); w.g12i = T(0);
  w.g21r = T(0);   w.g21i = T(0); w.g22r = T(0.5); w.g22i = T(0);
  al = unit_vec<4, T>(u);
  if (al > T(0)) {
    const T ur = u[0], ui = u[1], vr = u[2], vi = u[3];                     // u1 = H01/r, u2 = H02/r
    const T pr = fmaT(ur, br, -ui * bi), pi = fmaT(ur, bi, ui * br);        // u1 H12
    const T reP = fmaT(pr, vr, pi * vi);                                    // Re(u1 H12 u2*)
    s1 = fmaT(fmaT(ur, ur, ui * ui), d1, fmaT(fmaT(vr, vr, vi * vi), d2, reP + reP));
    s2 = (d1 + d2) - s1;
    const T dd = d2 - d1;
    const T uvr = fmaT(ur, vr, -ui * vi), uvi = fmaT(ur, vi, ui * vr);      // u1 u2
    const T u2r = fmaT(ur, ur, -ui * ui), u2i = T(2) * ur * ui;             // u1²
    const T v2r = fmaT(vr, vr, -vi * vi), v2i = T(2) * vr * vi;             // u2²
    const T xr = fmaT(uvr, dd, fmaT(u2r, br, -u2i * bi));
    const T xi = fmaT(uvi, dd, fmaT(u2r, bi, u2i * br));
    b12r = fmaT(-v2r, br, fmaT(-v2i, bi, xr));                              // − u2² H12*  (H12* = br − i bi)
    b12i = fmaT(-v2i, br, fmaT(v2r, bi, xi));
    const T h = T(0.5);
    w.g11r = h * ur;   w.g11i = -h * ui;         // H01*/r
    w.g21r = h * vr;   w.g21i = -h * vi;         // H02*/r
    w.g12r = -h * vr;  w.g12i = -h * vi;         // −H02/r
    w.g22r = h * ur;   w.g22i = h * ui;          // H01/r
  }
  T q[2] = {b12r, b12i};
  be = unit_vec<2, T>(q);
  if (be > T(0)) {                               // column 2 of g times e^{iψ} = B12*/|B12|
    const T er = q[0], ei = -q[1];
    const T x12r = fmaT(w.g12r, er, -w.g12i * ei), x12i = fmaT(w.g12r, ei, w.g12i * er);
    const T x22r = fmaT(w.g22r, er, -w.g22i * ei), x22i = fmaT(w.g22r, ei, w.g22i * er);
    w.g12r = x12r; w.g12i = x12i; w.g22r = x22r; w.g22i = x22i;
  }
}

// T₀ − I for T₀ = e^{−iD/2} e^{−iX} e^{−iD/2}, D = diag(s)/n, X = tridiagonal (al, be)/n, in the scaled form (2x, −2y)
// that sym_square_s carries.  Taylor branch as trotter_init (T₀ − I = −iA − A²/2 below taylor_bound); otherwise
// T₀_ij = e_i E_ij e_j with e_i = e^{−is_i/2}, E = e^{−iX} = I − iσX + K X² (σ = sin ρ/ρ, K = (cos ρ − 1)/ρ²,
// ρ² = al² + be²; X² = [[al², 0, al·be], [0, ρ², 0], [al·be, 0, be²]]).
template <typename T>
__device__ __forceinline__ void su3_init(const T* a, int tau, Sym3<T>& m, Su3W<T>& w) {
  T s0, s1, s2, al, be;
  su3_tridiagonalise<T>(a, s0, s1, s2, al, be, w);
  const T inv_n = ldexp(T(1), -tau);
  s0 *= inv_n; s1 *= inv_n; s2 *= inv_n; al *= inv_n; be *= inv_n;
  if ((fabs(s0) + fabs(s1) + fabs(s2) + T(2) * (al + be)) <= taylor_bound<T>()) {
    // (2x, −2y) = (−A², 2A), A = S/n:  A² = [[s0² + al², al(s0 + s1), al·be], [·, s1² + al² + be², be(s1 + s2)],
    // [·, ·, s2² + be²]]
    const T al2 = al * al, be2 = be * be;
    m.r00 = -fmaT(s0, s0, al2);         m.i00 = s0 + s0;
    m.r11 = -fmaT(s1, s1, al2 + be2);   m.i11 = s1 + s1;
    m.r22 = -fmaT(s2, s2, be2);         m.i22 = s2 + s2;
    m.r01 = -(al * (s0 + s1));          m.i01 = al + al;
    m.r12 = -(be * (s1 + s2));          m.i12 = be + be;
    m.r02 = -(al * be);                 m.i02 = T(0);
    return;
  }
  T sh[3], ch[3];
  const T sd[3] = {s0, s1, s2};
  const T big = fmax(fmax(fabs(s0), fabs(s1)), fabs(s2));
  if (big <= T(1.9073486328125e-06)) {          // half-angles ≤ 2^-20 (as trotter_init)
#pragma unroll
    for (int i = 0; i < 3; ++i) sincos_tiny<T>(sd[i] * T(0.5), &sh[i], &ch[i]);
  } else if (big <= T(0.03125)) {                // half-angles ≤ 2^-6: polynomial
#pragma unroll
    for (int i = 0; i < 3; ++i) sincos_small<T>(sd[i] * T(0.5), &sh[i], &ch[i]);
  } else {
#pragma unroll
    for (int i = 0; i < 3; ++i) sincosT(sd[i] * T(0.5), &sh[i], &ch[i]);
  }
  T sg, K;
  sinc_cosm1<T>(fmaT(al, al, be * be), &sg, &K);
  const T Ed[3] = {K * al * al, K * fmaT(al, al, be * be), K * be * be};      // E_ii − 1
  T dr[3], di[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {                  // e_i² E_ii − 1 = (v − i s2)(1 + E) + E, v − i s2 = expm1(−is_i)
    const T v = T(-2) * sh[i] * sh[i], s2i = T(2) * sh[i] * ch[i];
    dr[i] = fmaT(v, Ed[i], v + Ed[i]);
    di[i] = -s2i * (T(1) + Ed[i]);
  }
  // e_i e_j = (c_ij, −s_ij), c_ij = cos((s_i + s_j)/2), s_ij = sin((s_i + s_j)/2)
  const T c01 = fmaT(ch[0], ch[1], -sh[0] * sh[1]), s01 = fmaT(sh[0], ch[1], ch[0] * sh[1]);
  const T c12 = fmaT(ch[1], ch[2], -sh[1] * sh[2]), s12 = fmaT(sh[1], ch[2], ch[1] * sh[2]);
  const T c02 = fmaT(ch[0], ch[2], -sh[0] * sh[2]), s02 = fmaT(sh[0], ch[2], ch[0] * sh[2]);
  const T xa = sg * al, xb = sg * be, kab = K * al * be;
  // scaled: real parts ×2, imaginary parts ×(−2)
  m.r00 = T(2) * dr[0];  m.i00 = T(-2) * di[0];
  m.r11 = T(2) * dr[1];  m.i11 = T(-2) * di[1];
  m.r22 = T(2) * dr[2];  m.i22 = T(-2) * di[2];
  m.r01 = T(-2) * xa * s01;  m.i01 = T(2) * xa * c01;      // (c − is)(−iσal) = σal(−s − ic)
  m.r12 = T(-2) * xb * s12;  m.i12 = T(2) * xb * c12;
  m.r02 = T(2) * kab * c02;  m.i02 = T(2) * kab * s02;     // (c − is) K al be
}

// e = W (T₀^n − I) W† from the scaled symmetric residual (x̃, ỹ): Z̃ = x̃ − iỹ = 2(T₀^n − I), and g in w already
// carries the ½, so e = diag(½, g/2)·Z̃·diag(1, g)†.  24 complex multiply-adds.
template <typename T>
__device__ __forceinline__ void su3_expand(const Sym3<T>& m, const Su3W<T>& w, Res<3, T>& e) {
  // z_ij = (m.rij, −m.iij)
  const T z01r = m.r01, z01i = -m.i01, z02r = m.r02, z02i = -m.i02;
  const T z11r = m.r11, z11i = -m.i11, z12r = m.r12, z12i = -m.i12, z22r = m.r22, z22i = -m.i22;
  // full g = 2·(w) for the right factor g†
  const T G11r = T(2) * w.g11r, G11i = T(2) * w.g11i, G12r = T(2) * w.g12r, G12i = T(2) * w.g12i;
  const T G21r = T(2) * w.g21r, G21i = T(2) * w.g21i, G22r = T(2) * w.g22r, G22i = T(2) * w.g22i;
  e.re[0] = T(0.5) * m.r00;  e.im[0] = T(-0.5) * m.i00;
  // row 0: M0j = ½ Σ_k z0k conj(G_jk)
  const T hz01r = T(0.5) * z01r, hz01i = T(0.5) * z01i, hz02r = T(0.5) * z02r, hz02i = T(0.5) * z02i;
  e.re[1] = fmaT(hz01r, G11r, fmaT(hz01i, G11i, fmaT(hz02r, G12r, hz02i * G12i)));
  e.im[1] = fmaT(hz01i, G11r, fmaT(-hz01r, G11i, fmaT(hz02i, G12r, -hz02r * G12i)));
  e.re[2] = fmaT(hz01r, G21r, fmaT(hz01i, G21i, fmaT(hz02r, G22r, hz02i * G22i)));
  e.im[2] = fmaT(hz01i, G21r, fmaT(-hz01r, G21i, fmaT(hz02i, G22r, -hz02r * G22i)));
  // column 0: Mj0 = Σ_k (g_jk/2) zk0
  e.re[3] = fmaT(w.g11r, z01r, fmaT(-w.g11i, z01i, fmaT(w.g12r, z02r, -w.g12i * z02i)));
  e.im[3] = fmaT(w.g11r, z01i, fmaT(w.g11i, z01r, fmaT(w.g12r, z02i, w.g12i * z02r)));
  e.re[6] = fmaT(w.g21r, z01r, fmaT(-w.g21i, z01i, fmaT(w.g22r, z02r, -w.g22i * z02i)));
  e.im[6] = fmaT(w.g21r, z01i, fmaT(w.g21i, z01r, fmaT(w.g22r, z02i, w.g22i * z02r)));
  // block: N = (g/2) Zb, Mb = N g†
  const T n11r = fmaT(w.g11r, z11r, fmaT(-w.g11i, z11i, fmaT(w.g12r, z12r, -w.g12i * z12i)));
  const T n11i = fmaT(w.g11r, z11i, fmaT(w.g11i, z11r, fmaT(w.g12r, z12i, w.g12i * z12r)));
  const T n12r = fmaT(w.g11r, z12r, fmaT(-w.g11i, z12i, fmaT(w.g12r, z22r, -w.g12i * z22i)));
  const T n12i = fmaT(w.g11r, z12i, fmaT(w.g11i, z12r, fmaT(w.g12r, z22i, w.g12i * z22r)));
  const T n21r = fmaT(w.g21r, z11r, fmaT(-w.g21i, z11i, fmaT(w.g22r, z12r, -w.g22i * z12i)));
  const T n21i = fmaT(w.g21r, z11i, fmaT(w.g21i, z11r, fmaT(w.g22r, z12i, w.g22i * z12r)));
  const T n22r = fmaT(w.g21r, z12r, fmaT(-w.g21i, z12i, fmaT(w.g22r, z22r, -w.g22i * z22i)));
  const T n22i = fmaT(w.g21r, z12i, fmaT(w.g21i, z12r, fmaT(w.g22r, z22i, w.g22i * z22r)));
  // M_jl = N_j1 conj(G_l1) + N_j2 conj(G_l2)
  e.re[4] = fmaT(n11r, G11r, fmaT(n11i, G11i, fmaT(n12r, G12r, n12i * G12i)));
  e.im[4] = fmaT(n11i, G11r, fmaT(-n11r, G11i, fmaT(n12i, G12r, -n12r * G12i)));
  e.re[5] = fmaT(n11r, G21r, fmaT(n11i, G21i, fmaT(n12r, G22r, n12i * G22i)));
  e.im[5] = fmaT(n11i, G21r, fmaT(-n11r, G21i, fmaT(n12i, G22r, -n12r * G22i)));
  e.re[7] = fmaT(n21r, G11r, fmaT(n21i, G11i, fmaT(n22r, G12r, n22i * G12i)));
  e.im[7] = fmaT(n21i, G11r, fmaT(-n21r, G11i, fmaT(n22i, G12r, -n22r * G12i)));
  e.re[8] = fmaT(n21r, G21r, fmaT(n21i, G21i, fmaT(n22r, G22r, n22i * G22i)));
  e.im[8] = fmaT(n21i, G21r, fmaT(-n21r, G21i, fmaT(n22i, G22r, -n22r * G22i)));
}

template <typename T> __device__ __forceinline__ void trotter_residual_su3(const T* a, int tau, Res<3, T>& e) {
  Sym3<T> m;
  Su3W<T> w;
  su3_init<T>(a, tau, m, w);
  lt_square_tau<T>(m, tau);
  su3_expand<T>(m, w, e);
}

template <int SPIN, int EXPO, typename T> struct Expo;
// run(a, τ, e, series): the series choice (the caller's per-interval bound on r, see expo_su2) only matters for the
// SU(2) closed form.
template <int EXPO, typename T> struct Expo<SPIN_HALF, EXPO, T> {
  __device__ __forceinline__ static void run(const T a[4], int, Res<2, T>& e, int ser = 0) { expo_su2<T>(a, e, ser); }
};
template <typename T> struct Expo<SPIN_ONE, EXP_LIE_TROTTER, T> {
  __device__ __forceinline__ static void run(const T a[4], int tau, Res<3, T>& e, int = 0) {
    trotter_residual<T>(a, tau, e);
  }
};
template <typename T> struct Expo<SPIN_ONE, EXP_LIE_TROTTER_SU3, T> {
  __device__ __forceinline__ static void run(const T* a, int tau, Res<3, T>& e, int = 0) {
    trotter_residual_su3<T>(a, tau, e);
  }
};
template <typename T> __device__ __forceinline__ void expo_spin1_analytic(const T a[4], Res<3, T>& e) {
  Res<2, T> u;
  expo_su2<T>(a, u);
  su2_to_spin1<T>(u, e);
}
// The analytic spin-one path accumulates in SU(2) and maps once: D¹ is a homomorphism, so D¹(u_L)⋯D¹(u_1) =
// D¹(u_L⋯u_1) — the same interval operator, exactly (DESIGN.md §5 item 11).  Expo returns the SU(2) residual.
template <typename T> struct Expo<SPIN_ONE, EXP_ANALYTIC, T> {
  __device__ __forceinline__ static void run(const T a[4], int, Res<2, T>& e, int ser = 0) { expo_su2<T>(a, e, ser); }
};

// Dimension of the residual the interval kernel accumulates: 2 (SU(2) form) for spin-half and for the analytic
// spin-one exponentiator, 3 otherwise.
template <int SPIN, int EXPO> struct AccDim {
  static constexpr int D = (SPIN == SPIN_HALF || EXPO == EXP_ANALYTIC) ? 2 : 3;
};
template <typename T> __device__ __forceinline__ void acc_to_dim(const Res<2, T>& a, Res<2, T>& o) { o = a; }
template <typename T> __device__ __forceinline__ void acc_to_dim(const Res<2, T>& a, Res<3, T>& o) { su2_to_spin1<T>(a, o); }
template <typename T> __device__ __forceinline__ void acc_to_dim(const Res<3, T>& a, Res<3, T>& o) { o = a; }

}  // namespace ssb
