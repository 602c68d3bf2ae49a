// ops.cuh — the operator types the interval kernel's run aggregates and the state scans share (row a9).
//
// M is either CM<D> (a dense D×D complex matrix, the public U_k layout: W = D² complex128 in memory) or SU<D> (the
// SU(2) element (a, b) of U = [[a, b], [−b*, a*]]: W = 2 complex128, acting on a dim-D state directly (D = 2) or
// through D¹ (D = 3, reading R14)).  Combine = matrix product later·earlier (Eq. integration_compilation).
#pragma once

#include "spinsim_device.cuh"

namespace ssb {

template <int D> struct CM {  // dense complex matrix in registers
  double re[D * D], im[D * D];
  static constexpr int SD = D, W = D * D;   // state dimension, double2 per operator in memory
};

template <int D> __device__ __forceinline__ void cm_eye(CM<D>& m) {
#pragma unroll
  for (int e = 0; e < D * D; ++e) { m.re[e] = (e % (D + 1) == 0) ? 1.0 : 0.0; m.im[e] = 0.0; }
}

// c = a·b
template <int D> __device__ __forceinline__ CM<D> cm_mul(const CM<D>& a, const CM<D>& b) {
  CM<D> c;
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      double r = 0.0, m = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) {
        r = fma(a.re[i * D + k], b.re[k * D + j], r);
        r = fma(-a.im[i * D + k], b.im[k * D + j], r);
        m = fma(a.re[i * D + k], b.im[k * D + j], m);
        m = fma(a.im[i * D + k], b.re[k * D + j], m);
      }
      c.re[i * D + j] = r;
      c.im[i * D + j] = m;
    }
  return c;
}

// y = a·x
template <int D> __device__ __forceinline__ void cm_apply(const CM<D>& a, const double xr[D], const double xi[D],
                                                          double yr[D], double yi[D]) {
#pragma unroll
  for (int i = 0; i < D; ++i) {
    double r = 0.0, m = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      r = fma(a.re[i * D + k], xr[k], r);
      r = fma(-a.im[i * D + k], xi[k], r);
      m = fma(a.re[i * D + k], xi[k], m);
      m = fma(a.im[i * D + k], xr[k], m);
    }
    yr[i] = r;
    yi[i] = m;
  }
}

template <int D> __device__ __forceinline__ void cm_load(const double2* src, CM<D>& m) {
#pragma unroll
  for (int e = 0; e < D * D; ++e) { const double2 v = src[e]; m.re[e] = v.x; m.im[e] = v.y; }
}
template <int D> __device__ __forceinline__ void cm_load_cg(const double2* src, CM<D>& m) {
#pragma unroll
  for (int e = 0; e < D * D; ++e) { const double2 v = __ldcg(src + e); m.re[e] = v.x; m.im[e] = v.y; }
}
template <int D> __device__ __forceinline__ void cm_store(double2* dst, const CM<D>& m) {
#pragma unroll
  for (int e = 0; e < D * D; ++e) dst[e] = make_double2(m.re[e], m.im[e]);
}
template <int D> __device__ __forceinline__ CM<D> cm_shfl_up(const CM<D>& m, int delta) {
  CM<D> r;
#pragma unroll
  for (int e = 0; e < D * D; ++e) {
    r.re[e] = __shfl_up_sync(0xffffffffu, m.re[e], delta);
    r.im[e] = __shfl_up_sync(0xffffffffu, m.im[e], delta);
  }
  return r;
}

template <int D> __device__ __forceinline__ CM<D> cm_shfl_down(const CM<D>& m, int delta) {
  CM<D> r;
#pragma unroll
  for (int e = 0; e < D * D; ++e) {
    r.re[e] = __shfl_down_sync(0xffffffffu, m.re[e], delta);
    r.im[e] = __shfl_down_sync(0xffffffffu, m.im[e], delta);
  }
  return r;
}
template <int D> __device__ __forceinline__ CM<D> cm_shfl_idx(const CM<D>& m, int src) {
  CM<D> r;
#pragma unroll
  for (int e = 0; e < D * D; ++e) {
    r.re[e] = __shfl_sync(0xffffffffu, m.re[e], src);
    r.im[e] = __shfl_sync(0xffffffffu, m.im[e], src);
  }
  return r;
}

// ---- compact SU(2) operators -------------------------------------------------------------------------------------
// U = [[a, b], [−b*, a*]] held as (a, b): every operator of the spin-half path is in SU(2) (DESIGN.md §5 item 10),
// and the analytic spin-one operator is D¹ of one (reading R14, §5 item 11), so the products of the scan stay in
// SU(2) exactly (group law) and only the action on a state depends on D: directly for D = 2, through
// D¹(U) = [[a², √2ab, b²], [−√2ab*, |a|²−|b|², √2a*b], [b*², −√2a*b*, a*²]] for D = 3.
template <int D> struct SU {
  double ar, ai, br, bi;
  static constexpr int SD = D, W = 2;
};
template <int D> __device__ __forceinline__ void cm_eye(SU<D>& m) { m.ar = 1.0; m.ai = m.br = m.bi = 0.0; }
// x·y = (x_a y_a − x_b y_b*, x_a y_b + x_b y_a*)
template <int D> __device__ __forceinline__ SU<D> cm_mul(const SU<D>& x, const SU<D>& y) {
  SU<D> c;
  c.ar = fma(x.ar, y.ar, fma(-x.ai, y.ai, fma(-x.br, y.br, -(x.bi * y.bi))));
  c.ai = fma(x.ar, y.ai, fma(x.ai, y.ar, fma(-x.bi, y.br, x.br * y.bi)));
  c.br = fma(x.ar, y.br, fma(-x.ai, y.bi, fma(x.br, y.ar, x.bi * y.ai)));
  c.bi = fma(x.ar, y.bi, fma(x.ai, y.br, fma(x.bi, y.ar, -(x.br * y.ai))));
  return c;
}
template <int D> __device__ __forceinline__ void cm_apply(const SU<D>& u, const double xr[D], const double xi[D],
                                                          double yr[D], double yi[D]) {
  if constexpr (D == 2) {
    // y0 = a x0 + b x1,  y1 = −b* x0 + a* x1
    yr[0] = fma(u.ar, xr[0], fma(-u.ai, xi[0], fma(u.br, xr[1], -(u.bi * xi[1]))));
    yi[0] = fma(u.ar, xi[0], fma(u.ai, xr[0], fma(u.br, xi[1], u.bi * xr[1])));
    yr[1] = fma(-u.br, xr[0], fma(-u.bi, xi[0], fma(u.ar, xr[1], u.ai * xi[1])));
    yi[1] = fma(-u.br, xi[0], fma(u.bi, xr[0], fma(u.ar, xi[1], -(u.ai * xr[1]))));
  } else {
    // D¹ entries from a, b (the map of the interval kernel's su2_to_spin1, full rather than residual form)
    const double a2r = u.ar * u.ar - u.ai * u.ai, a2i = 2.0 * u.ar * u.ai;             // a²
    const double b2r = u.br * u.br - u.bi * u.bi, b2i = 2.0 * u.br * u.bi;             // b²
    const double abr = kSqrt2 * (u.ar * u.br - u.ai * u.bi), abi = kSqrt2 * (u.ar * u.bi + u.ai * u.br);   // √2ab
    const double acr = kSqrt2 * (u.ar * u.br + u.ai * u.bi), aci = kSqrt2 * (u.ar * u.bi - u.ai * u.br);   // √2a*b
    const double dd = (u.ar * u.ar + u.ai * u.ai) - (u.br * u.br + u.bi * u.bi);      // |a|² − |b|²
    // row 0: a² x0 + √2ab x1 + b² x2
    yr[0] = fma(a2r, xr[0], fma(-a2i, xi[0], fma(abr, xr[1], fma(-abi, xi[1], fma(b2r, xr[2], -(b2i * xi[2]))))));
    yi[0] = fma(a2r, xi[0], fma(a2i, xr[0], fma(abr, xi[1], fma(abi, xr[1], fma(b2r, xi[2], b2i * xr[2])))));
    // row 1: −√2ab* x0 + (|a|²−|b|²) x1 + √2a*b x2, with −√2ab* = −conj(√2a*b)
    yr[1] = fma(-acr, xr[0], fma(-aci, xi[0], fma(dd, xr[1], fma(acr, xr[2], -(aci * xi[2])))));
    yi[1] = fma(-acr, xi[0], fma(aci, xr[0], fma(dd, xi[1], fma(acr, xi[2], aci * xr[2]))));
    // row 2: b*² x0 − √2a*b* x1 + a*² x2, with √2a*b* = conj(√2ab)
    yr[2] = fma(b2r, xr[0], fma(b2i, xi[0], fma(-abr, xr[1], fma(-abi, xi[1], fma(a2r, xr[2], a2i * xi[2])))));
    yi[2] = fma(b2r, xi[0], fma(-b2i, xr[0], fma(-abr, xi[1], fma(abi, xr[1], fma(a2r, xi[2], -(a2i * xr[2]))))));
  }
}
template <int D> __device__ __forceinline__ void cm_load(const double2* src, SU<D>& m) {
  const double2 a = src[0], b = src[1];
  m.ar = a.x; m.ai = a.y; m.br = b.x; m.bi = b.y;
}
template <int D> __device__ __forceinline__ void cm_load_cg(const double2* src, SU<D>& m) {
  const double2 a = __ldcg(src), b = __ldcg(src + 1);
  m.ar = a.x; m.ai = a.y; m.br = b.x; m.bi = b.y;
}
template <int D> __device__ __forceinline__ void cm_store(double2* dst, const SU<D>& m) {
  dst[0] = make_double2(m.ar, m.ai);
  dst[1] = make_double2(m.br, m.bi);
}
template <int D> __device__ __forceinline__ SU<D> cm_shfl_up(const SU<D>& m, int delta) {
  SU<D> r;
  r.ar = __shfl_up_sync(0xffffffffu, m.ar, delta); r.ai = __shfl_up_sync(0xffffffffu, m.ai, delta);
  r.br = __shfl_up_sync(0xffffffffu, m.br, delta); r.bi = __shfl_up_sync(0xffffffffu, m.bi, delta);
  return r;
}
template <int D> __device__ __forceinline__ SU<D> cm_shfl_down(const SU<D>& m, int delta) {
  SU<D> r;
  r.ar = __shfl_down_sync(0xffffffffu, m.ar, delta); r.ai = __shfl_down_sync(0xffffffffu, m.ai, delta);
  r.br = __shfl_down_sync(0xffffffffu, m.br, delta); r.bi = __shfl_down_sync(0xffffffffu, m.bi, delta);
  return r;
}
template <int D> __device__ __forceinline__ SU<D> cm_shfl_idx(const SU<D>& m, int src) {
  SU<D> r;
  r.ar = __shfl_sync(0xffffffffu, m.ar, src); r.ai = __shfl_sync(0xffffffffu, m.ai, src);
  r.br = __shfl_sync(0xffffffffu, m.br, src); r.bi = __shfl_sync(0xffffffffu, m.bi, src);
  return r;
}

// ⟨J⟩ = (Re ψ†Jxψ, Re ψ†Jyψ, ψ†Jzψ), closed forms of the textbook matrices (reading R5).
template <int D> __device__ __forceinline__ void spin_of(const double pr[D], const double pi[D], double j[3]) {
  if (D == 2) {
    // Jx = σx/2: Re(ψ0*ψ1); Jy = σy/2: Im(ψ0*ψ1); Jz = (|ψ0|² − |ψ1|²)/2
    j[0] = pr[0] * pr[1] + pi[0] * pi[1];
    j[1] = pr[0] * pi[1] - pi[0] * pr[1];
    j[2] = 0.5 * ((pr[0] * pr[0] + pi[0] * pi[0]) - (pr[1] * pr[1] + pi[1] * pi[1]));
  } else {
    // Jx = (1/√2)·tridiag(1): √2 Re(ψ0*ψ1 + ψ1*ψ2); Jy: √2 Im(ψ0*ψ1 + ψ1*ψ2); Jz = |ψ0|² − |ψ2|²
    j[0] = kSqrt2 * (pr[0] * pr[1] + pi[0] * pi[1] + pr[1] * pr[D - 1] + pi[1] * pi[D - 1]);
    j[1] = kSqrt2 * (pr[0] * pi[1] - pi[0] * pr[1] + pr[1] * pi[D - 1] - pi[1] * pr[D - 1]);
    j[2] = (pr[0] * pr[0] + pi[0] * pi[0]) - (pr[D - 1] * pr[D - 1] + pi[D - 1] * pi[D - 1]);
  }
}

}  // namespace ssb
