// spinsim_oracle.cpp — the CPU ORACLE for the Spinsim hot path (arXiv 2204.05586).
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs may load this library.  The product path (paper_2204_05586_b200/) never
// links, imports or calls it, and it shares no code, header or constant generator with the CUDA path.
//
// What it is: a plain, slow, obviously-correct transcription of the paper's algorithm, step by step, in
// the paper's order and notation.  Every function cites the PAPER.md passage ("P:<line>", section/equation)
// it follows.  The readings adopted where the paper is silent or garbled are listed in DESIGN.md §3 and
// referenced here as "reading Rn".
//
// Precision: templated on the real type R.  R = long double (x87, 64-bit mantissa) is the PARITY
// reference; R = double is the instantiation timed as the CPU baseline.  Compile with
// -ffp-contract=off so the FP64 time-grid formulas (reading R7) are evaluated exactly as written.
//
// Plain (non-residual) accumulation U_r <- u·U_r — the residual trick is used only where the paper
// itself prescribes it: inside the Lie–Trotter exponentiator.
//
// Parity status of each function is stated in DESIGN.md §4 ("pins"); every function below is pinned by
// a `-m "not gpu"` test in tests/test_oracle_pins.py.

#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>
#include <atomic>

namespace oracle {

// ------------------------------------------------------------------------------------------------
// Enumerations (the oracle's own; the Python side maps names -> these numbers).
// ------------------------------------------------------------------------------------------------
enum Spin { HALF = 1, ONE = 2 };                            // 2j
enum Method { CF4 = 0, MIDPOINT = 1, HEUN = 2 };
enum Expo { ANALYTIC = 0, LIE_TROTTER = 1, LIE_TROTTER_SU3 = 2 };   // P:359; general su(3): P:478-479
enum Field { CONSTANT = 0, RABI_LINEAR = 1, RABI_CIRCULAR = 2, NEURAL = 3, GRADIENT = 4,
             SU3_CONSTANT = 6, SU3_DRIVE = 7 };                     // 6, 7: general spin-one

// Field samples carry NF = 8 coefficients (ωx, ωy, ωz, ωq, ωu1, ωu2, ωv1, ωv2) of
// H = ωx Jx + ωy Jy + ωz Jz + ωq Q + ωu1 U1 + ωu2 U2 + ωv1 V1 + ωv2 V2; the last four are zero for
// every field of the 4-operator family and are used only by the su(3) exponentiator.
constexpr int NF = 8;

template <class R> using Cx = std::complex<R>;

template <class R> struct Mat {               // dense dim x dim complex matrix, dim in {2, 3}
  int n = 0;
  Cx<R> a[3][3];
  static Mat eye(int n) { Mat m; m.n = n; for (int i = 0; i < n; ++i) m.a[i][i] = R(1); return m; }
  static Mat zero(int n) { Mat m; m.n = n; return m; }
};

template <class R> Mat<R> mul(const Mat<R>& x, const Mat<R>& y) {   // plain triple loop
  Mat<R> z = Mat<R>::zero(x.n);
  for (int i = 0; i < x.n; ++i)
    for (int j = 0; j < x.n; ++j) {
      Cx<R> s = 0;
      for (int k = 0; k < x.n; ++k) s += x.a[i][k] * y.a[k][j];
      z.a[i][j] = s;
    }
  return z;
}

// ------------------------------------------------------------------------------------------------
// Time grid — reading R7: the paper fixes t_k = t_0 + Δt·k and δt = Δt/L
// but not their floating-point evaluation.  Both sides evaluate them in IEEE double, exactly as below,
// so the sample times are bit-identical; all further arithmetic is in R.
// ------------------------------------------------------------------------------------------------
struct Grid {
  double t0, dt_out, dt_int;   // t_0, Δt, δt (δt := Δt / L)
  long long K, L;
};

// Gauss–Legendre offsets g1,2 = ½(1 ∓ 1/√3), evaluated in long double and rounded once to
// double.  The pins check they are the correctly-rounded doubles.
inline double gauss_g1() { return (double)((1.0L - 1.0L / std::sqrt(3.0L)) / 2.0L); }
inline double gauss_g2() { return (double)((1.0L + 1.0L / std::sqrt(3.0L)) / 2.0L); }

inline double grid_tk(const Grid& g, long long k) {     // t_k = fl(t0 + fl(k·Δt))
  volatile double kd = (double)k * g.dt_out;
  return g.t0 + kd;
}
inline double grid_off(const Grid& g, long long l, double frac) {   // off = fl(fl(l·δt) + fl(frac·δt))
  volatile double a = (double)l * g.dt_int;
  volatile double b = frac * g.dt_int;
  return a + b;
}

// ------------------------------------------------------------------------------------------------
// Field functions (P:131-183 parametrisation; built-ins replacing the user's numba function).
// Sample time is the unrounded pair (t_k, off) — reading R8: phases are formed from ((R)t_k + off) in R.
// ------------------------------------------------------------------------------------------------
template <class R> R sinp(R x) {                  // "a single cycle of a sine wave", reading R12
  const R two_pi = R(2) * std::acos(R(-1));
  return (x >= R(0) && x <= two_pi) ? std::sin(x) : R(0);
}

template <class R> void field_sample(int field, const double* p, double t_k, double off, R f[NF]) {
  const R t = (R)t_k + (R)off;
  for (int j = 0; j < NF; ++j) f[j] = R(0);
  switch (field) {
    case CONSTANT:         // p = [ωx, ωy, ωz, ωq]
      f[0] = p[0]; f[1] = p[1]; f[2] = p[2]; f[3] = p[3];
      break;
    case RABI_LINEAR:      // p = [ω0, Ω]; H = ω0 Jz + 2Ω cos(ω0 t) Jx  (the paper's drive form)
      f[0] = R(2) * (R)p[1] * std::cos((R)p[0] * t);
      f[2] = p[0];
      break;
    case RABI_CIRCULAR:    // p = [ω0, Ω]; H = ω0 Jz + Ω(cos(ω0 t) Jx + sin(ω0 t) Jy)   (exact Rabi pin)
      f[0] = (R)p[1] * std::cos((R)p[0] * t);
      f[1] = (R)p[1] * std::sin((R)p[0] * t);
      f[2] = p[0];
      break;
    case NEURAL: {         // Eq. neural_pulse: H = ω Jz + 2Ω cos(ω t) Jx + Ω_p sinp(Ω(t − t_p)) Jz
      // p = [ω_bias, ω_rf, Ω, Ω_p, ω_sig, t_p, ω_q] (ω split into bias/RF, Ω into dressing/signal freq;
      // ω_q: quadratic shift Q term, P:178 — reading R15).
      f[0] = R(2) * (R)p[2] * std::cos((R)p[1] * t);
      const R pulse_arg = (R)p[4] * (((R)t_k - (R)p[5]) + (R)off);
      f[2] = (R)p[0] + (R)p[3] * sinp(pulse_arg);
      f[3] = p[6];
      break;
    }
    case GRADIENT:         // MRI example: ω_z = x − 2y, p = [x, y]
      f[2] = (R)p[0] - R(2) * (R)p[1];
      break;
    case SU3_CONSTANT:     // p = all 8 coefficients, constant in time
      for (int j = 0; j < NF; ++j) f[j] = p[j];
      break;
    case SU3_DRIVE: {      // reading R20: bias + quadratic shift + a circular drive of frequency ω_d coupling the
      // upper and lower pairs with different strengths (Ω_x Jφ + Ω_v Vφ) and a two-photon drive (Ω_u Uφ) at 2ω_d
      // ("different coupling between the lower and upper pairs of states, or with two-photon coupling").
      // p = [ω0, ω_q, Ω_x, Ω_v, Ω_u, ω_d]
      const R ph = (R)p[5] * t;
      f[0] = (R)p[2] * std::cos(ph);          f[1] = (R)p[2] * std::sin(ph);
      f[2] = p[0];                            f[3] = p[1];
      f[4] = (R)p[4] * std::cos(R(2) * ph);   f[5] = (R)p[4] * std::sin(R(2) * ph);
      f[6] = (R)p[3] * std::cos(ph);          f[7] = (R)p[3] * std::sin(ph);
      break;
    }
  }
}

inline int field_num_params(int field) {
  switch (field) {
    case CONSTANT: return 4;
    case RABI_LINEAR: return 2;
    case RABI_CIRCULAR: return 2;
    case NEURAL: return 7;
    case GRADIENT: return 2;
    case SU3_CONSTANT: return 8;
    case SU3_DRIVE: return 6;
  }
  return -1;
}

// ------------------------------------------------------------------------------------------------
// Rotating frame (§rotating_frame): H_r = R(t)(ωx Jx + ωy Jy)R(−t) + (ωz − ω_r)Jz + ωq Q with
// R(t) = exp(i ω_r Jz t).  Since exp(iθJz) Jx exp(−iθJz) = cosθ Jx − sinθ Jy and
// exp(iθJz) Jy exp(−iθJz) = cosθ Jy + sinθ Jx, the transverse coefficients rotate as below
// (pinned by explicit matrix conjugation in the tests).  t_local = 0 at the interval start (reading R6).
// ------------------------------------------------------------------------------------------------
//
// General spin-one (reading R19/R20): conjugation multiplies matrix entry (i, j) by e^{iθ(m_i − m_j)}, so the
// Δm = ±1 quadrupole pair (V1, V2) rotates like (Jx, Jy) and the Δm = ±2 pair (U1, U2) by the angle 2θ.
template <class R> void to_rotating_frame(R f[NF], R t_local, R omega_r) {
  const R th = omega_r * t_local;
  const R c = std::cos(th), s = std::sin(th);
  const R fx = f[0], fy = f[1];
  f[0] = c * fx + s * fy;
  f[1] = -s * fx + c * fy;
  f[2] = f[2] - omega_r;
  // f[3] (ωq) unchanged: [Jz, Q] = 0
  const R c2 = std::cos(R(2) * th), s2 = std::sin(R(2) * th);
  const R u1 = f[4], u2 = f[5];
  f[4] = c2 * u1 + s2 * u2;
  f[5] = -s2 * u1 + c2 * u2;
  const R v1 = f[6], v2 = f[7];
  f[6] = c * v1 + s * v2;
  f[7] = -s * v1 + c * v2;
}

// ------------------------------------------------------------------------------------------------
// Exponentiators: exp(−i(ax Jx + ay Jy + az Jz + aq Q)), a = h·δt (reading R2).
// ------------------------------------------------------------------------------------------------

// Spin-half analytic form: with r = |a|, exp(−i a·σ/2) = cos(r/2) I − i (sin(r/2)/r)(a·σ).
template <class R> Mat<R> expm_su2(R ax, R ay, R az) {
  Mat<R> U = Mat<R>::zero(2);
  const R r = std::sqrt(ax * ax + ay * ay + az * az);
  const R c = std::cos(r / R(2));
  const R s = (r == R(0)) ? R(0.5) : std::sin(r / R(2)) / r;     // reading R4
  const Cx<R> I(0, 1);
  U.a[0][0] = c - I * s * az;
  U.a[0][1] = -I * s * Cx<R>(ax, -ay);
  U.a[1][0] = -I * s * Cx<R>(ax, ay);
  U.a[1][1] = c + I * s * az;
  return U;
}

// expm1(iθ) = e^{iθ} − 1 without cancellation: (cosθ − 1) + i sinθ = −2 sin²(θ/2) + i sinθ.
template <class R> Cx<R> expm1i(R th) {
  const R sh = std::sin(th / R(2));
  return Cx<R>(-R(2) * sh * sh, std::sin(th));
}

// Leapfrog factor T − I (Eq. lie_trotter_4, with the two misprinted entries corrected —
// reading R1: T22 = cosΦ e^{i2q/3}, T13 = −(sin(Φ/2) e^{−iq/6} e^{−iφ})²), arguments already divided by
// n (z = az/n, q = aq/n, Φ = √(ax²+ay²)/n, φ = atan2(ay, ax)).  Diagonal computed with expm1-style
// kernels instead of subtracting 1.  Basis order m = +1, 0, −1 (reading R5).
template <class R> Mat<R> trotter_factor_residual(R Phi, R phi, R z, R q) {
  Mat<R> a = Mat<R>::zero(3);
  const Cx<R> I(0, 1);
  const R rt2 = std::sqrt(R(2));
  const R c = std::cos(Phi / R(2)), s = std::sin(Phi / R(2));
  const Cx<R> em_phi = std::exp(-I * phi);                // e^{−iφ}
  const Cx<R> ep_phi = std::exp(I * phi);                 // e^{+iφ}
  const Cx<R> ez_m = std::exp(-I * z / R(2));             // e^{−iz/2}
  const Cx<R> ez_p = std::exp(I * z / R(2));              // e^{+iz/2}
  const Cx<R> eq6_p = std::exp(I * q / R(6));             // e^{+iq/6}
  const Cx<R> eq6_m = std::exp(-I * q / R(6));            // e^{−iq/6}
  const R sinPhi = std::sin(Phi);
  // Off-diagonal entries, as printed in Eq. lie_trotter_4 except T13 (reading R1).
  a.a[0][1] = (-I / rt2) * sinPhi * eq6_p * ez_m * em_phi;
  a.a[0][2] = -((s * eq6_m * em_phi) * (s * eq6_m * em_phi));
  a.a[1][0] = (-I / rt2) * sinPhi * eq6_p * ez_m * ep_phi;
  a.a[1][2] = (-I / rt2) * sinPhi * eq6_p * ez_p * em_phi;
  a.a[2][0] = -((s * eq6_m * ep_phi) * (s * eq6_m * ep_phi));
  a.a[2][1] = (-I / rt2) * sinPhi * eq6_p * ez_p * ep_phi;
  // Diagonal minus identity.
  //   T11 = (c e^{−iz/2} e^{−iq/6})² = c² e^{−iθ1},  θ1 = z + q/3:  T11 − 1 = expm1(−iθ1) − s² e^{−iθ1}
  //   T22 = cosΦ e^{i2q/3} = (1 − 2s²) e^{iθ2}, θ2 = 2q/3:         T22 − 1 = expm1(iθ2) − 2s² e^{iθ2}
  //   T33 = (c e^{iz/2} e^{−iq/6})² = c² e^{iθ3}, θ3 = z − q/3:     T33 − 1 = expm1(iθ3) − s² e^{iθ3}
  (void)c;
  const R th1 = z + q / R(3), th2 = R(2) * q / R(3), th3 = z - q / R(3);
  a.a[0][0] = expm1i(-th1) - s * s * std::exp(-I * th1);
  a.a[1][1] = expm1i(th2) - R(2) * s * s * std::exp(I * th2);
  a.a[2][2] = expm1i(th3) - s * s * std::exp(I * th3);
  return a;
}

// One residual squaring: with T = I + a, T² − I = (a + 2I) a.
template <class R> Mat<R> residual_square(const Mat<R>& a) {
  Mat<R> b = a;
  for (int i = 0; i < 3; ++i) b.a[i][i] += R(2);          // a + 2I
  return mul(b, a);                                      // (a + 2I) a
}

// Lie–Trotter exponentiator: U = T^n, n = 2^τ, by τ residual squarings s = (a + 2I)a
// (P:456-462), then the identity is added back.
template <class R> Mat<R> expm_lie_trotter(R ax, R ay, R az, R aq, int tau) {
  const R n = std::ldexp(R(1), tau);
  const R Phi = std::sqrt(ax * ax + ay * ay) / n;
  const R phi = std::atan2(ay, ax);                        // atan2(0,0) = 0: reading R3
  const R z = az / n, q = aq / n;
  Mat<R> a = trotter_factor_residual(Phi, phi, z, q);
  for (int it = 0; it < tau; ++it) a = residual_square(a);
  for (int i = 0; i < 3; ++i) a.a[i][i] += R(1);
  return a;
}

// "Analytic" spin-one exponential (reading R14; not in the paper): the spin-1 representation D¹ of the
// SU(2) closed form, exact iff ωq = 0.  For U = [[α, β], [−β*, α*]]:
//   D¹(U) = [[α², √2αβ, β²], [−√2αβ*, |α|²−|β|², √2α*β], [β*², −√2α*β*, α*²]].
template <class R> Mat<R> expm_spin1_analytic(R ax, R ay, R az) {
  const Mat<R> u = expm_su2(ax, ay, az);
  const Cx<R> al = u.a[0][0], be = u.a[0][1];
  const R rt2 = std::sqrt(R(2));
  Mat<R> D = Mat<R>::zero(3);
  D.a[0][0] = al * al;
  D.a[0][1] = rt2 * al * be;
  D.a[0][2] = be * be;
  D.a[1][0] = -rt2 * al * std::conj(be);
  D.a[1][1] = std::norm(al) - std::norm(be);
  D.a[1][2] = rt2 * std::conj(al) * be;
  D.a[2][0] = std::conj(be) * std::conj(be);
  D.a[2][1] = -rt2 * std::conj(al) * std::conj(be);
  D.a[2][2] = std::conj(al) * std::conj(al);
  return D;
}

// ------------------------------------------------------------------------------------------------
// General spin-one exponentiator (the paper ships it but does not describe it — readings
// R19, R20 in DESIGN.md).  H = Σ a_j A_j over the su(3) basis of P:184-187, in the order of Eq.:
//   A_0..A_3 = Jx, Jy, Jz (reading R5), Q = diag(1,−2,1)/3;
//   A_4..A_7 = U1 = Jx² − Jy², U2 = JxJy + JyJx (Δm = ±2), V1 = JxJz + JzJx, V2 = JyJz + JzJy (Δm = ±1)   (R19),
// multiplied out below from the spin matrices themselves.
// Lie–Trotter exactly as the paper prints it: T is the product of the exponentials of the single basis
// elements, exp(−i a_j A_j / n), each of which "has a known analytic form" — taken in the leapfrog
// (symmetric) arrangement the paper applies to its own factor (e^{−iD/2} … e^{−iD/2}, D = the diagonal
// operators outermost), reading R20:
//   T = E_2 E_3 E_4 E_5 E_6 E_7 E_0 · e^{−i a_1 A_1/n} · E_0 E_7 E_6 E_5 E_4 E_3 E_2,   E_j = exp(−i a_j A_j / 2n).
// Closed form of one factor exp(−iθA) − I (residual):
//   diagonal A (Jz, Q): entrywise expm1(−iθλ_i);
//   A³ = A (Jx, Jy, U1, U2, V1, V2 — eigenvalues 0, ±1): −i sinθ A + (cosθ − 1) A², cosθ − 1 = −2 sin²(θ/2).
// The residuals are multiplied by (I + x)(I + y) − I = x + y + xy, then τ residual squarings s = (a + 2I)a
// and the identity added back.
// ------------------------------------------------------------------------------------------------
template <class R> Mat<R> res_prod(const Mat<R>& x, const Mat<R>& y) {   // (I + x)(I + y) − I
  Mat<R> z = mul(x, y);
  for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) z.a[i][j] += x.a[i][j] + y.a[i][j];
  return z;
}

template <class R> struct SpinOneBasis {
  Mat<R> A[NF];     // Jx, Jy, Jz, Q, U1, U2, V1, V2
};

template <class R> SpinOneBasis<R> spin_one_basis() {
  const Cx<R> I(0, 1);
  const R s = R(1) / std::sqrt(R(2));
  Mat<R> Jx = Mat<R>::zero(3), Jy = Mat<R>::zero(3), Jz = Mat<R>::zero(3), Q = Mat<R>::zero(3);
  Jx.a[0][1] = Jx.a[1][0] = Jx.a[1][2] = Jx.a[2][1] = s;
  Jy.a[0][1] = -I * s; Jy.a[1][0] = I * s; Jy.a[1][2] = -I * s; Jy.a[2][1] = I * s;
  Jz.a[0][0] = R(1); Jz.a[2][2] = R(-1);
  Q.a[0][0] = R(1) / R(3); Q.a[1][1] = R(-2) / R(3); Q.a[2][2] = R(1) / R(3);
  auto anti = [](const Mat<R>& x, const Mat<R>& y) {       // x y + y x
    Mat<R> a = mul(x, y), b = mul(y, x);
    for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) a.a[i][j] += b.a[i][j];
    return a;
  };
  Mat<R> U1 = mul(Jx, Jx), Jy2 = mul(Jy, Jy);
  for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) U1.a[i][j] -= Jy2.a[i][j];
  SpinOneBasis<R> b;
  b.A[0] = Jx; b.A[1] = Jy; b.A[2] = Jz; b.A[3] = Q;
  b.A[4] = U1; b.A[5] = anti(Jx, Jy); b.A[6] = anti(Jx, Jz); b.A[7] = anti(Jy, Jz);
  return b;
}

// exp(−iθA) − I for one basis element A, closed forms above.
template <class R> Mat<R> basis_factor_residual(const Mat<R>& A, bool diagonal, R th) {
  Mat<R> e = Mat<R>::zero(3);
  if (diagonal) {
    for (int i = 0; i < 3; ++i) e.a[i][i] = expm1i(-th * A.a[i][i].real());
    return e;
  }
  const Cx<R> I(0, 1);
  const R sh = std::sin(th / R(2));
  const R cosm1 = -R(2) * sh * sh, sn = std::sin(th);
  const Mat<R> A2 = mul(A, A);
  for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) e.a[i][j] = -I * sn * A.a[i][j] + cosm1 * A2.a[i][j];
  return e;
}

// T − I of the leapfrog basis product, arguments a[8] divided by n.
template <class R> Mat<R> trotter_factor_residual_su3(const R a[NF], R n) {
  static const SpinOneBasis<R> B = spin_one_basis<R>();     // built once (thread-safe static initialisation)
  const int outer[7] = {2, 3, 4, 5, 6, 7, 0};     // D = (Jz, Q) outermost as in P:374, then U, V, Jx; Jy in the middle
  const int middle = 1;
  auto factor = [&](int j, R frac) { return basis_factor_residual(B.A[j], j == 2 || j == 3, frac * a[j] / n); };
  Mat<R> t = Mat<R>::zero(3);
  for (int q = 0; q < 7; ++q) t = res_prod(t, factor(outer[q], R(0.5)));
  t = res_prod(t, factor(middle, R(1)));
  for (int q = 6; q >= 0; --q) t = res_prod(t, factor(outer[q], R(0.5)));
  return t;
}

template <class R> Mat<R> expm_lie_trotter_su3(const R a[NF], int tau) {
  const R n = std::ldexp(R(1), tau);
  Mat<R> m = trotter_factor_residual_su3(a, n);
  for (int it = 0; it < tau; ++it) m = residual_square(m);
  for (int i = 0; i < 3; ++i) m.a[i][i] += R(1);
  return m;
}

template <class R> Mat<R> exponentiate(int spin, int expo, int tau, const R a[NF]) {
  if (spin == HALF) return expm_su2(a[0], a[1], a[2]);
  if (expo == LIE_TROTTER) return expm_lie_trotter(a[0], a[1], a[2], a[3], tau);
  if (expo == LIE_TROTTER_SU3) return expm_lie_trotter_su3(a, tau);
  return expm_spin1_analytic(a[0], a[1], a[2]);
}

// ------------------------------------------------------------------------------------------------
// Dense Taylor scaling-and-squaring exponential exp(−i s H) — used ONLY by the pins (a library-style
// reference independent of the structured exponentiators above).
// ------------------------------------------------------------------------------------------------
template <class R> Mat<R> expm_dense(const Mat<R>& H, R s) {
  const int n = H.n;
  Mat<R> A = Mat<R>::zero(n);
  const Cx<R> mi(0, -1);
  R norm1 = 0;
  for (int j = 0; j < n; ++j) {
    R col = 0;
    for (int i = 0; i < n; ++i) { A.a[i][j] = mi * s * H.a[i][j]; col += std::abs(A.a[i][j]); }
    if (col > norm1) norm1 = col;
  }
  int sq = 0;
  while (norm1 > R(1) / R(32)) { norm1 /= 2; ++sq; }
  const R scale = std::ldexp(R(1), -sq);
  for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) A.a[i][j] *= scale;
  Mat<R> E = Mat<R>::eye(n), term = Mat<R>::eye(n);
  for (int k = 1; k <= 24; ++k) {
    term = mul(term, A);
    for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) term.a[i][j] /= R(k);
    for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) E.a[i][j] += term.a[i][j];
  }
  for (int k = 0; k < sq; ++k) E = mul(E, E);
  return E;
}

// ------------------------------------------------------------------------------------------------
// One fine step u_l (P:324-341 for CF4; P:702-704 for the Euler samplers, readings R13).
// ------------------------------------------------------------------------------------------------
struct Config {
  int spin, method, expo, tau, frame, field;
};

template <class R> void sample_in_frame(const Config& c, const double* p, double t_k, double off,
                                        R omega_r, R f[NF]) {
  field_sample<R>(c.field, p, t_k, off, f);
  if (c.frame) to_rotating_frame<R>(f, (R)off, omega_r);       // applied at each sample
}

template <class R> Mat<R> fine_step(const Config& c, const Grid& g, const double* p, double t_k,
                                    long long l, R omega_r) {
  const R dt = (R)g.dt_int;
  if (c.method == CF4) {
    // Sample times t1,2 = t + ½(1 ∓ 1/√3)δt.
    const double off1 = grid_off(g, l, gauss_g1());
    const double off2 = grid_off(g, l, gauss_g2());
    R f1[NF], f2[NF];
    sample_in_frame<R>(c, p, t_k, off1, omega_r, f1);
    sample_in_frame<R>(c, p, t_k, off2, omega_r, f2);
    // Weights (3 ± 2√3)/12 (Eqs. cf4_sample_1/2).
    const R wp = (R(3) + R(2) * std::sqrt(R(3))) / R(12);
    const R wm = (R(3) - R(2) * std::sqrt(R(3))) / R(12);
    R a1[NF], a2[NF];
    for (int j = 0; j < NF; ++j) {
      a1[j] = (wp * f1[j] + wm * f2[j]) * dt;   // H̄1 δt
      a2[j] = (wm * f1[j] + wp * f2[j]) * dt;   // H̄2 δt
    }
    const Mat<R> e1 = exponentiate<R>(c.spin, c.expo, c.tau, a1);
    const Mat<R> e2 = exponentiate<R>(c.spin, c.expo, c.tau, a2);
    return mul(e2, e1);                          // exp(−iH̄2δt) exp(−iH̄1δt)  (Eq. cf4_implementation)
  }
  R f[NF];
  if (c.method == MIDPOINT) {                    // "modified Euler": one sample at t + δt/2
    sample_in_frame<R>(c, p, t_k, grid_off(g, l, 0.5), omega_r, f);
  } else {                                       // HEUN, "improved Euler": average of H(t), H(t+δt)
    R fa[NF], fb[NF];
    sample_in_frame<R>(c, p, t_k, grid_off(g, l, 0.0), omega_r, fa);
    sample_in_frame<R>(c, p, t_k, grid_off(g, l + 1, 0.0), omega_r, fb);
    for (int j = 0; j < NF; ++j) f[j] = (fa[j] + fb[j]) / R(2);
  }
  R a[NF];
  for (int j = 0; j < NF; ++j) a[j] = f[j] * dt;
  return exponentiate<R>(c.spin, c.expo, c.tau, a);
}

// ------------------------------------------------------------------------------------------------
// Interval operator U_k (§parallelization; Fig. architecture; frame P:539-545).
// ------------------------------------------------------------------------------------------------
// Frame rate of interval k: ω_r = ω_z(t_k + Δt/2) from the lab field, 0 with the frame off.
template <class R> R frame_omega(const Config& c, const Grid& g, const double* p, double t_k) {
  if (!c.frame) return R(0);
  R f[NF];
  field_sample<R>(c.field, p, t_k, 0.5 * g.dt_out, f);
  return f[2];
}

template <class R> Mat<R> interval_operator(const Config& c, const Grid& g, const double* p, long long k) {
  const int dim = (c.spin == HALF) ? 2 : 3;
  const double t_k = grid_tk(g, k);
  const R omega_r = frame_omega<R>(c, g, p, t_k);
  Mat<R> U = Mat<R>::eye(dim);                   // U_r initialised to the identity
  for (long long l = 0; l < g.L; ++l) {
    const Mat<R> u = fine_step<R>(c, g, p, t_k, l, omega_r);
    U = mul(u, U);                               // u premultiplied to U_r
  }
  if (c.frame) {                                 // U_k = R_{ω_r}(−Δt) U_k^r = exp(−iω_r Jz Δt) U_k^r
    const Cx<R> I(0, 1);
    for (int i = 0; i < dim; ++i) {
      const R m = (dim == 2) ? (i == 0 ? R(0.5) : R(-0.5)) : R(1 - i);
      const Cx<R> ph = std::exp(-I * omega_r * m * (R)g.dt_out);
      for (int j = 0; j < dim; ++j) U.a[i][j] *= ph;
    }
  }
  return U;
}

// ------------------------------------------------------------------------------------------------
// Advisory Magnus-convergence diagnostic (the Magnus series of a step converges if ∫‖H‖₂ < ξ ≈ 1.08686870).
// Per fine step: δt·(‖H(t₁)‖₂ + ‖H(t₂)‖₂)/2, the two-point Gauss–Legendre estimate of ∫‖H‖₂ on the CF4 sample times,
// with H the field in the integration frame; the result is the maximum over the sweep.  H is assembled as the
// dense matrix Σ f_j A_j from the operator DEFINITIONS (spin-half: σ/2; spin-one: Jx, Jy, Jz, Q and the quadrupoles
// U1 = Jx² − Jy², U2 = {Jx, Jy}, V1 = {Jx, Jz}, V2 = {Jy, Jz} of reading R19, multiplied out in spin_one_basis), and ‖H‖₂ is the
// largest |eigenvalue|, from the roots of the characteristic polynomial.
// ------------------------------------------------------------------------------------------------
template <class R> Mat<R> dense_hamiltonian(int spin, const R f[NF]) {
  if (spin == HALF) {
    Mat<R> h = Mat<R>::zero(2);
    h.a[0][0] = f[2] / R(2);                 h.a[1][1] = -f[2] / R(2);
    h.a[0][1] = Cx<R>(f[0], -f[1]) / R(2);   h.a[1][0] = Cx<R>(f[0], f[1]) / R(2);
    return h;
  }
  static const SpinOneBasis<R> B = spin_one_basis<R>();
  Mat<R> h = Mat<R>::zero(3);
  for (int j = 0; j < NF; ++j)
    for (int r = 0; r < 3; ++r) for (int c = 0; c < 3; ++c) h.a[r][c] += f[j] * B.A[j].a[r][c];
  return h;
}

template <class R> R spectral_norm(const Mat<R>& h) {
  if (h.n == 2) {   // λ = (tr ± √(tr² − 4 det))/2 (real for Hermitian h)
    const R tr = (h.a[0][0] + h.a[1][1]).real();
    const R det = (h.a[0][0] * h.a[1][1] - h.a[0][1] * h.a[1][0]).real();
    const R disc = std::sqrt(std::max(R(0), tr * tr - R(4) * det));
    return std::max(std::fabs((tr + disc) / R(2)), std::fabs((tr - disc) / R(2)));
  }
  // λ = μ + tr/3 with μ the roots of μ³ − pμ − q, B = h − (tr/3)I, p = tr(B²)/2, q = det B (trigonometric form)
  const R m = (h.a[0][0] + h.a[1][1] + h.a[2][2]).real() / R(3);
  Mat<R> B = h;
  for (int i = 0; i < 3; ++i) B.a[i][i] -= m;
  const Mat<R> B2 = mul(B, B);
  const R p = (B2.a[0][0] + B2.a[1][1] + B2.a[2][2]).real() / R(2);
  const R q = (B.a[0][0] * (B.a[1][1] * B.a[2][2] - B.a[1][2] * B.a[2][1]) -
               B.a[0][1] * (B.a[1][0] * B.a[2][2] - B.a[1][2] * B.a[2][0]) +
               B.a[0][2] * (B.a[1][0] * B.a[2][1] - B.a[1][1] * B.a[2][0])).real();
  if (!(p > R(0))) return std::fabs(m);
  const R r = R(2) * std::sqrt(p / R(3));
  const R c = std::min(R(1), std::max(R(-1), (R(3) * q / (R(2) * p)) * std::sqrt(R(3) / p)));
  const R phi = std::acos(c) / R(3), two_pi_3 = R(2) * std::acos(R(-1)) / R(3);
  R best = 0;
  for (int k = 0; k < 3; ++k) best = std::max(best, std::fabs(r * std::cos(phi - two_pi_3 * k) + m));
  return best;
}

template <class R> R magnus_bound(const Config& c, const Grid& g, const double* p) {
  R worst = 0;
  for (long long k = 0; k < g.K; ++k) {
    const double t_k = grid_tk(g, k);
    const R omega_r = frame_omega<R>(c, g, p, t_k);
    for (long long l = 0; l < g.L; ++l) {
      R f1[NF], f2[NF];
      sample_in_frame<R>(c, p, t_k, grid_off(g, l, gauss_g1()), omega_r, f1);
      sample_in_frame<R>(c, p, t_k, grid_off(g, l, gauss_g2()), omega_r, f2);
      const R n = (R)g.dt_int * (spectral_norm(dense_hamiltonian<R>(c.spin, f1)) +
                                 spectral_norm(dense_hamiltonian<R>(c.spin, f2))) / R(2);
      worst = std::max(worst, n);
    }
  }
  return worst;
}

// Validation and planning: K = (t1−t0)/Δt and L = Δt/δt must be integral (reading R10).
inline int plan(double t0, double t1, double dt_int, double dt_out, long long* K, long long* L, double* dt) {
  if (!(t1 > t0) || !(dt_int > 0) || !(dt_out > 0)) return -1;
  const double kf = (t1 - t0) / dt_out;
  const double lf = dt_out / dt_int;
  const long long k = std::llround(kf), l = std::llround(lf);
  if (k < 1 || l < 1) return -1;
  if (std::fabs(kf - (double)k) > 1e-9 * kf || std::fabs(lf - (double)l) > 1e-9 * lf) return -1;
  *K = k; *L = l; *dt = dt_out / (double)l;
  return 0;
}

template <class R> void store(const Mat<R>& U, double* out) {
  for (int i = 0; i < U.n; ++i)
    for (int j = 0; j < U.n; ++j) {
      out[2 * (i * U.n + j)] = (double)U.a[i][j].real();
      out[2 * (i * U.n + j) + 1] = (double)U.a[i][j].imag();
    }
}

// Full evaluation: U[b][k] for k in [k_begin, k_end) in parallel over (b, k) with std::thread (the paper's
// CPU-parallel mode), then the sequential chain ψ_{k+1} = U_k ψ_k per sweep (Eq.
// integration_compilation; chained on the CPU as in P:640).  The chain is carried in R.
template <class R>
int evaluate(const Config& c, const Grid& g, long long batch, const double* sweep, int n_params,
             const double* psi0, double* states, double* unitaries, int nthreads,
             long long k_begin, long long k_end) {
  const int dim = (c.spin == HALF) ? 2 : 3;
  const long long nk = k_end - k_begin;
  std::vector<Mat<R>> U((size_t)(batch * nk));
  std::atomic<long long> next(0);
  const long long total = batch * nk;
  auto worker = [&]() {
    for (;;) {
      const long long id = next.fetch_add(1);
      if (id >= total) break;
      const long long b = id / nk, k = k_begin + id % nk;
      U[(size_t)id] = interval_operator<R>(c, g, sweep + b * n_params, k);
    }
  };
  if (nthreads <= 0) nthreads = (int)std::thread::hardware_concurrency();
  if (nthreads < 1) nthreads = 1;
  std::vector<std::thread> pool;
  for (int t = 0; t < nthreads; ++t) pool.emplace_back(worker);
  for (auto& th : pool) th.join();
  for (long long b = 0; b < batch; ++b) {
    Cx<R> psi[3];
    for (int i = 0; i < dim; ++i) psi[i] = Cx<R>((R)psi0[b * 2 * dim + 2 * i], (R)psi0[b * 2 * dim + 2 * i + 1]);
    double* sb = states ? states + b * (nk + 1) * 2 * dim : nullptr;
    if (sb) for (int i = 0; i < dim; ++i) { sb[2 * i] = (double)psi[i].real(); sb[2 * i + 1] = (double)psi[i].imag(); }
    for (long long kk = 0; kk < nk; ++kk) {
      const Mat<R>& Uk = U[(size_t)(b * nk + kk)];
      if (unitaries) store(Uk, unitaries + (b * nk + kk) * 2 * dim * dim);
      Cx<R> nxt[3];
      for (int i = 0; i < dim; ++i) {
        nxt[i] = 0;
        for (int j = 0; j < dim; ++j) nxt[i] += Uk.a[i][j] * psi[j];
      }
      for (int i = 0; i < dim; ++i) psi[i] = nxt[i];
      if (sb) {
        double* o = sb + (kk + 1) * 2 * dim;
        for (int i = 0; i < dim; ++i) { o[2 * i] = (double)psi[i].real(); o[2 * i + 1] = (double)psi[i].imag(); }
      }
    }
  }
  return 0;
}

}  // namespace oracle

// ==================================================================================================
// C ABI for the Python test harness (oracle/__init__.py).  All I/O is double / interleaved complex128.
// `use_ld` selects the long-double (parity) or double (timing) instantiation.
// ==================================================================================================
using namespace oracle;

static bool valid_config(const Config& c) {
  if (c.spin != HALF && c.spin != ONE) return false;
  if (c.method < CF4 || c.method > HEUN) return false;
  if (c.expo != ANALYTIC && c.expo != LIE_TROTTER && c.expo != LIE_TROTTER_SU3) return false;
  if (c.spin == HALF && c.expo != ANALYTIC) return false;
  // fields with U/V components need the su(3) exponentiator (the others would drop them)
  if ((c.field == SU3_CONSTANT || c.field == SU3_DRIVE) && c.expo != LIE_TROTTER_SU3) return false;
  if (c.tau < 0 || c.tau > 60) return false;
  if (field_num_params(c.field) < 0) return false;
  return true;
}

extern "C" {

int oracle_constants(double* out) {        // [g1, g2, w+, w−] as doubles
  out[0] = gauss_g1();
  out[1] = gauss_g2();
  out[2] = (double)((3.0L + 2.0L * std::sqrt(3.0L)) / 12.0L);
  out[3] = (double)((3.0L - 2.0L * std::sqrt(3.0L)) / 12.0L);
  return 0;
}

int oracle_num_params(int field) { return field_num_params(field); }

int oracle_plan(double t0, double t1, double dt_int, double dt_out, long long* K, long long* L, double* dt) {
  return plan(t0, t1, dt_int, dt_out, K, L, dt);
}

int oracle_grid(double t0, double dt_out, double dt_int, long long k, long long l, double* out) {
  Grid g{t0, dt_out, dt_int, 0, 0};
  out[0] = grid_tk(g, k);
  out[1] = grid_off(g, l, gauss_g1());
  out[2] = grid_off(g, l, gauss_g2());
  out[3] = grid_off(g, l, 0.5);
  return 0;
}

// out: [8] (ωx, ωy, ωz, ωq, ωu1, ωu2, ωv1, ωv2)
int oracle_field_sample(int field, const double* p, double t_k, double off, int use_ld, double* out) {
  if (field_num_params(field) < 0) return -1;
  if (use_ld) { long double f[NF]; field_sample<long double>(field, p, t_k, off, f); for (int j = 0; j < NF; ++j) out[j] = (double)f[j]; }
  else { double f[NF]; field_sample<double>(field, p, t_k, off, f); for (int j = 0; j < NF; ++j) out[j] = f[j]; }
  return 0;
}

// f_in, out: [8]
int oracle_rotating_frame(const double* f_in, double t_local, double omega_r, double* out) {
  long double f[NF];
  for (int j = 0; j < NF; ++j) f[j] = f_in[j];
  to_rotating_frame<long double>(f, t_local, omega_r);
  for (int j = 0; j < NF; ++j) out[j] = (double)f[j];
  return 0;
}

// args: [n][na] (ax, ay, az, aq[, au1, au2, av1, av2]), na = 4 or 8; out: [n][dim][dim] complex128
int oracle_exponentiate(int spin, int expo, int tau, int use_ld, long long n, int na, const double* args,
                        double* out) {
  Config c{spin, CF4, expo, tau, 0, CONSTANT};
  if (!valid_config(c) || (na != 4 && na != NF)) return -1;
  const int dim = (spin == HALF) ? 2 : 3;
  for (long long i = 0; i < n; ++i) {
    if (use_ld) {
      long double a[NF] = {};
      for (int j = 0; j < na; ++j) a[j] = args[na * i + j];
      store(exponentiate<long double>(spin, expo, tau, a), out + i * 2 * dim * dim);
    } else {
      double a[NF] = {};
      for (int j = 0; j < na; ++j) a[j] = args[na * i + j];
      store(exponentiate<double>(spin, expo, tau, a), out + i * 2 * dim * dim);
    }
  }
  return 0;
}

// T − I of the general spin-one leapfrog basis product (reading R20) for a[8] divided by n = 2^tau (long double).
int oracle_trotter_residual_su3(const double* a, int tau, double* out) {
  long double al[NF];
  for (int j = 0; j < NF; ++j) al[j] = a[j];
  store(trotter_factor_residual_su3<long double>(al, std::ldexp(1.0L, tau)), out);
  return 0;
}

// T − I of the leapfrog factor for given (Φ, φ, z, q) (already divided by n), long double.
int oracle_trotter_residual(double Phi, double phi, double z, double q, double* out) {
  store(trotter_factor_residual<long double>(Phi, phi, z, q), out);
  return 0;
}

// exp(−i s H) for a dense Hermitian H [dim][dim] complex128 (pins only).
int oracle_expm_dense(int dim, const double* H, double s, double* out) {
  if (dim != 2 && dim != 3) return -1;
  Mat<long double> h = Mat<long double>::zero(dim);
  for (int i = 0; i < dim; ++i)
    for (int j = 0; j < dim; ++j) h.a[i][j] = Cx<long double>(H[2 * (i * dim + j)], H[2 * (i * dim + j) + 1]);
  store(expm_dense<long double>(h, s), out);
  return 0;
}

int oracle_fine_step(int spin, int method, int expo, int tau, int frame, int field, int use_ld,
                     double t0, double dt_out, double dt_int, const double* p, long long k, long long l,
                     double omega_r, double* out) {
  Config c{spin, method, expo, tau, frame, field};
  if (!valid_config(c)) return -1;
  Grid g{t0, dt_out, dt_int, 0, 0};
  const double t_k = grid_tk(g, k);
  if (use_ld) store(fine_step<long double>(c, g, p, t_k, l, omega_r), out);
  else store(fine_step<double>(c, g, p, t_k, l, omega_r), out);
  return 0;
}

int oracle_evaluate(int spin, int method, int expo, int tau, int frame, int field, int use_ld,
                    double t0, double t1, double dt_int, double dt_out,
                    long long batch, const double* sweep, const double* psi0,
                    double* states, double* unitaries, int nthreads,
                    long long k_begin, long long k_end) {
  Config c{spin, method, expo, tau, frame, field};
  if (!valid_config(c) || batch < 0) return -1;
  Grid g{t0, dt_out, 0, 0, 0};
  if (plan(t0, t1, dt_int, dt_out, &g.K, &g.L, &g.dt_int) != 0) return -1;
  if (k_end < 0) k_end = g.K;
  if (k_begin < 0 || k_end > g.K || k_begin >= k_end) return -1;
  const int np = field_num_params(field);
  if (use_ld) return evaluate<long double>(c, g, batch, sweep, np, psi0, states, unitaries, nthreads, k_begin, k_end);
  return evaluate<double>(c, g, batch, sweep, np, psi0, states, unitaries, nthreads, k_begin, k_end);
}

// Sequential chain only (Eq. integration_compilation, as the paper's CPU loop P:640), long double:
// states[b][0] = psi0[b], states[b][k+1] = U[b][k] states[b][k].  Also returns the product A[b] = U[b][K−1]⋯U[b][0]
// (if `aggregate` is non-NULL) by plain left-multiplication in index order.
int oracle_chain(int dim, long long batch, long long K, const double* U, const double* psi0, double* states,
                 double* aggregate) {
  typedef long double R;
  for (long long b = 0; b < batch; ++b) {
    Cx<R> psi[3];
    for (int i = 0; i < dim; ++i) psi[i] = Cx<R>(psi0[(b * dim + i) * 2], psi0[(b * dim + i) * 2 + 1]);
    double* sb = states + b * (K + 1) * dim * 2;
    for (int i = 0; i < dim; ++i) { sb[2 * i] = (double)psi[i].real(); sb[2 * i + 1] = (double)psi[i].imag(); }
    Mat<R> A = Mat<R>::eye(dim);
    for (long long k = 0; k < K; ++k) {
      Mat<R> Uk = Mat<R>::zero(dim);
      const double* u = U + ((b * K + k) * dim * dim) * 2;
      for (int i = 0; i < dim; ++i)
        for (int j = 0; j < dim; ++j) Uk.a[i][j] = Cx<R>(u[2 * (i * dim + j)], u[2 * (i * dim + j) + 1]);
      Cx<R> nxt[3];
      for (int i = 0; i < dim; ++i) {
        nxt[i] = 0;
        for (int j = 0; j < dim; ++j) nxt[i] += Uk.a[i][j] * psi[j];
      }
      for (int i = 0; i < dim; ++i) psi[i] = nxt[i];
      double* o = sb + (k + 1) * dim * 2;
      for (int i = 0; i < dim; ++i) { o[2 * i] = (double)psi[i].real(); o[2 * i + 1] = (double)psi[i].imag(); }
      if (aggregate) A = mul(Uk, A);
    }
    if (aggregate) store(A, aggregate + b * dim * dim * 2);
  }
  return 0;
}

// Expected spin projection ⟨J⟩ = (ψ†Jxψ, ψ†Jyψ, ψ†Jzψ), long double.
int oracle_spin_projection(int spin, long long n, const double* states, double* out) {
  const int dim = (spin == HALF) ? 2 : 3;
  typedef long double R;
  const Cx<R> I(0, 1);
  Mat<R> J[3];
  for (int a = 0; a < 3; ++a) J[a] = Mat<R>::zero(dim);
  if (dim == 2) {                 // Pauli matrices halved
    J[0].a[0][1] = J[0].a[1][0] = R(0.5);
    J[1].a[0][1] = -I * R(0.5); J[1].a[1][0] = I * R(0.5);
    J[2].a[0][0] = R(0.5); J[2].a[1][1] = R(-0.5);
  } else {                        // spin-1 matrices, basis m = +1, 0, −1 (reading R5)
    const R h = R(1) / std::sqrt(R(2));
    J[0].a[0][1] = J[0].a[1][0] = J[0].a[1][2] = J[0].a[2][1] = h;
    J[1].a[0][1] = -I * h; J[1].a[1][0] = I * h; J[1].a[1][2] = -I * h; J[1].a[2][1] = I * h;
    J[2].a[0][0] = R(1); J[2].a[2][2] = R(-1);
  }
  for (long long s = 0; s < n; ++s) {
    Cx<R> psi[3];
    for (int i = 0; i < dim; ++i) psi[i] = Cx<R>(states[s * 2 * dim + 2 * i], states[s * 2 * dim + 2 * i + 1]);
    for (int a = 0; a < 3; ++a) {
      Cx<R> acc = 0;
      for (int i = 0; i < dim; ++i)
        for (int j = 0; j < dim; ++j) acc += std::conj(psi[i]) * J[a].a[i][j] * psi[j];
      out[3 * s + a] = (double)acc.real();
    }
  }
  return 0;
}

// Magnus diagnostic per sweep (long double); f_in: [8] field coefficients for a direct spectral-norm query.
int oracle_magnus_bound(int spin, int frame, int field, double t0, double t1, double dt_int, double dt_out,
                        long long batch, const double* sweep, double* out) {
  Config c{spin, CF4, spin == HALF ? ANALYTIC : LIE_TROTTER_SU3, 24, frame, field};
  if (field_num_params(field) < 0 || (spin != HALF && spin != ONE)) return -1;
  Grid g{t0, dt_out, 0, 0, 0};
  if (plan(t0, t1, dt_int, dt_out, &g.K, &g.L, &g.dt_int) != 0) return -1;
  const int np = field_num_params(field);
  for (long long b = 0; b < batch; ++b) out[b] = (double)magnus_bound<long double>(c, g, sweep + b * np);
  return 0;
}

int oracle_spectral_norm(int spin, const double* f_in, double* out) {
  long double f[NF];
  for (int j = 0; j < NF; ++j) f[j] = f_in[j];
  *out = (double)spectral_norm(dense_hamiltonian<long double>(spin, f));
  return 0;
}

// Eq. error: ε = (1/K) sqrt(Σ_k Σ_m |ψ − ψ_base|²), 1/K outside the root as printed (reading R18).
double oracle_rms_error(long long K, int dim, const double* a, const double* b) {
  long double acc = 0;
  for (long long i = 0; i < K * dim; ++i) {
    const long double dr = (long double)a[2 * i] - b[2 * i], di = (long double)a[2 * i + 1] - b[2 * i + 1];
    acc += dr * dr + di * di;
  }
  return (double)(std::sqrt(acc) / (long double)K);
}

}  // extern "C"
