// scan.cu — state propagation and the small kernels around it.
//
// ψ_{k+1} = U_k ψ_k (Eq. integration_compilation) is a linear recurrence; the paper runs it sequentially
// on the CPU.  Here it is an associative matrix-product scan (combine = later·earlier) over tiles of
// kTile consecutive intervals of one sweep, with decoupled look-back between tiles:
//   1. a block takes the next tile ticket (atomic; tiles of a sweep get increasing tickets, so every tile a block
//      waits on is already resident → forward progress), stages the tile's U_k in shared memory (coalesced),
//   2. each thread multiplies its kItems consecutive operators (thread aggregate), a warp Kogge–Stone scan with
//      shuffles and a block combine through shared memory give every thread its exclusive prefix and the block its
//      tile aggregate,
//   3. the tile publishes its aggregate (flag AGG), looks back over predecessors (M ← M·A_j′ over AGG tiles until a
//      PREFIX tile gives ψ_end(j′)), publishes its inclusive end state ψ_end = A·ψ_in (flag PREFIX),
//   4. each thread applies its exclusive prefix to ψ_in and then its own operators in order, writing states through
//      shared memory (coalesced).
// HBM traffic per interval: read U_k (2·dim² doubles) + write ψ_{k+1} (2·dim doubles) — 192 B (spin-one) /
// 96 B (spin-half): the kernel is HBM bound.
#include <cuda/atomic>

#include "kernels.h"

namespace ssb {

template <int D> struct ScanCfg;
template <> struct ScanCfg<2> { static constexpr int kItems = 4; };
template <> struct ScanCfg<3> { static constexpr int kItems = 2; };
constexpr int kScanThreads = 128;
template <int D> constexpr int tile_size() { return kScanThreads * ScanCfg<D>::kItems; }

enum { FLAG_EMPTY = 0, FLAG_AGG = 1, FLAG_PREFIX = 2 };

template <int D> struct CM {  // dense complex matrix in registers
  double re[D * D], im[D * D];
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

// Workspace layout (all offsets 256-byte aligned): [ticket u64][flags int32 × ntiles][agg dim² c128 × ntiles]
// [psi_end dim c128 × ntiles].
static inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

template <int D> struct ScanLayout {
  int64_t tiles_per_sweep, ntiles;
  size_t off_flags, off_agg, off_psi, total;
  ScanLayout(int64_t batch, int64_t k_count) {
    tiles_per_sweep = (k_count + tile_size<D>() - 1) / tile_size<D>();
    ntiles = batch * tiles_per_sweep;
    off_flags = 256;
    off_agg = align256(off_flags + sizeof(int) * (size_t)ntiles);
    off_psi = align256(off_agg + sizeof(double2) * D * D * (size_t)ntiles);
    total = align256(off_psi + sizeof(double2) * D * (size_t)ntiles);
  }
};

struct ScanArgs {
  int64_t batch, k_count, tiles_per_sweep;
  const double2* U;          // [batch][k_count][D][D]
  const double2* psi0;       // [batch][D]
  double2* states;           // [batch][k_count+1][D]  (SCAN mode)
  double2* aggregate_out;    // [ntiles][D][D]          (AGGREGATE mode: per-tile totals)
  unsigned long long* ticket;
  int* flags;
  double2* agg;
  double2* psi_end;
};

template <int D, bool SCAN>
__global__ void __launch_bounds__(kScanThreads) scan_kernel(const ScanArgs a) {
  constexpr int C = ScanCfg<D>::kItems;
  constexpr int TILE = kScanThreads * C;
  constexpr int NW = kScanThreads / 32;
  extern __shared__ double2 smem[];          // [TILE·D·D] operators, then [TILE·D] states (SCAN)
  double2* sU = smem;
  double2* sPsi = smem + TILE * D * D;
  __shared__ double2 sWarpTot[NW][D * D];
  __shared__ double2 sPsiIn[D];
  __shared__ long long sTicket;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) sTicket = (long long)atomicAdd(a.ticket, 1ull);
  __syncthreads();
  const long long ticket = sTicket;
  const long long b = ticket / a.tiles_per_sweep;
  const long long j = ticket - b * a.tiles_per_sweep;
  const long long k0 = j * TILE;
  const int n_items = (int)min((long long)TILE, a.k_count - k0);

  // 1. stage U (coalesced 16-byte loads, streaming)
  const double2* gU = a.U + ((size_t)b * a.k_count + k0) * D * D;
  for (int e = tid; e < n_items * D * D; e += kScanThreads) sU[e] = __ldcs(gU + e);
  __syncthreads();

  // 2. thread aggregate over its C consecutive items: P = U_{c+C−1} ⋯ U_c
  CM<D> P;
  cm_eye(P);
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const int it = tid * C + c;
    if (it < n_items) {
      CM<D> u;
      cm_load(sU + it * D * D, u);
      P = cm_mul(u, P);
    }
  }
  // warp inclusive scan (later·earlier)
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const CM<D> q = cm_shfl_up(P, off);
    if (lane >= off) P = cm_mul(P, q);
  }
  CM<D> E = cm_shfl_up(P, 1);  // exclusive within the warp
  if (lane == 0) cm_eye(E);
  if (lane == 31) cm_store(sWarpTot[warp], P);
  __syncthreads();
  // prefix of earlier warps W = T_{w−1} ⋯ T_0 ; thread exclusive X = E · W
  CM<D> W;
  cm_eye(W);
  for (int w = 0; w < warp; ++w) {
    CM<D> t;
    cm_load(sWarpTot[w], t);
    W = cm_mul(t, W);
  }
  const CM<D> X = cm_mul(E, W);

  if (tid == 0) {
    CM<D> tot;  // block aggregate T_{NW−1} ⋯ T_0
    cm_eye(tot);
    for (int w = 0; w < NW; ++w) {
      CM<D> t;
      cm_load(sWarpTot[w], t);
      tot = cm_mul(t, tot);
    }
    if (!SCAN) {
      cm_store(a.aggregate_out + (size_t)ticket * D * D, tot);
    } else {
      cuda::atomic_ref<int, cuda::thread_scope_device> my_flag(a.flags[ticket]);
      double pr[D], pi[D];
      if (j == 0) {
        for (int d = 0; d < D; ++d) { const double2 v = a.psi0[b * D + d]; pr[d] = v.x; pi[d] = v.y; }
      } else {
        // 3a. publish the aggregate
        cm_store(a.agg + (size_t)ticket * D * D, tot);
        my_flag.store(FLAG_AGG, cuda::memory_order_release);
        // 3b. look back
        CM<D> M;
        cm_eye(M);
        long long jj = ticket - 1;
        for (;;) {
          cuda::atomic_ref<int, cuda::thread_scope_device> f(a.flags[jj]);
          int fv;
          while ((fv = f.load(cuda::memory_order_acquire)) == FLAG_EMPTY) __nanosleep(20);
          if (fv == FLAG_PREFIX) {
            double er[D], ei[D];
            for (int d = 0; d < D; ++d) { const double2 v = __ldcg(a.psi_end + jj * D + d); er[d] = v.x; ei[d] = v.y; }
            cm_apply(M, er, ei, pr, pi);
            break;
          }
          CM<D> A;
          cm_load_cg(a.agg + (size_t)jj * D * D, A);
          M = cm_mul(M, A);
          --jj;
        }
      }
      // 3c. publish the inclusive end state ψ_end = tot·ψ_in
      double er[D], ei[D];
      cm_apply(tot, pr, pi, er, ei);
      for (int d = 0; d < D; ++d) a.psi_end[ticket * D + d] = make_double2(er[d], ei[d]);
      my_flag.store(FLAG_PREFIX, cuda::memory_order_release);
      for (int d = 0; d < D; ++d) sPsiIn[d] = make_double2(pr[d], pi[d]);
      if (j == 0)
        for (int d = 0; d < D; ++d) a.states[(size_t)b * (a.k_count + 1) * D + d] = make_double2(pr[d], pi[d]);
    }
  }
  if (!SCAN) return;
  __syncthreads();

  // 4. apply: ψ = X·ψ_in, then the thread's own operators in order
  double xr[D], xi[D], yr[D], yi[D];
#pragma unroll
  for (int d = 0; d < D; ++d) { xr[d] = sPsiIn[d].x; xi[d] = sPsiIn[d].y; }
  cm_apply(X, xr, xi, yr, yi);
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const int it = tid * C + c;
    if (it < n_items) {
      CM<D> u;
      cm_load(sU + it * D * D, u);
      cm_apply(u, yr, yi, xr, xi);
#pragma unroll
      for (int d = 0; d < D; ++d) { yr[d] = xr[d]; yi[d] = xi[d]; sPsi[it * D + d] = make_double2(xr[d], xi[d]); }
    }
  }
  __syncthreads();
  double2* gS = a.states + ((size_t)b * (a.k_count + 1) + k0 + 1) * D;
  for (int e = tid; e < n_items * D; e += kScanThreads) __stcs(gS + e, sPsi[e]);
}

// Per-sweep product of the tile aggregates, in order: A[b] = T_{n−1} ⋯ T_0.
template <int D>
__global__ void combine_tiles_kernel(int64_t batch, int64_t tiles_per_sweep, const double2* tiles, double2* out) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  CM<D> A;
  cm_eye(A);
  for (int64_t t = 0; t < tiles_per_sweep; ++t) {
    CM<D> T;
    cm_load(tiles + ((size_t)b * tiles_per_sweep + t) * D * D, T);
    A = cm_mul(T, A);
  }
  cm_store(out + (size_t)b * D * D, A);
}

// carry[b] = A_{part−1} ⋯ A_0 ψ0[b], applied to the state in increasing partition order.
template <int D>
__global__ void compose_carry_kernel(int64_t batch, int part, const double2* aggs, const double2* psi0, double2* carry) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  double xr[D], xi[D], yr[D], yi[D];
  for (int d = 0; d < D; ++d) { xr[d] = psi0[b * D + d].x; xi[d] = psi0[b * D + d].y; }
  for (int g = 0; g < part; ++g) {
    CM<D> A;
    cm_load(aggs + ((size_t)g * batch + b) * D * D, A);
    cm_apply(A, xr, xi, yr, yi);
    for (int d = 0; d < D; ++d) { xr[d] = yr[d]; xi[d] = yi[d]; }
  }
  for (int d = 0; d < D; ++d) carry[b * D + d] = make_double2(xr[d], xi[d]);
}

// ⟨J⟩ = (Re ψ†Jxψ, Re ψ†Jyψ, ψ†Jzψ), closed forms of the textbook matrices (reading R5).
template <int D>
__global__ void spin_projection_kernel(int64_t n, const double2* states, double* out) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  double2 p[D];
#pragma unroll
  for (int d = 0; d < D; ++d) p[d] = states[s * D + d];
  double jx, jy, jz;
  if (D == 2) {
    // Jx = σx/2: Re(ψ0*ψ1); Jy = σy/2: Im(ψ0*ψ1); Jz = (|ψ0|² − |ψ1|²)/2
    const double cr = p[0].x * p[1].x + p[0].y * p[1].y, ci = p[0].x * p[1].y - p[0].y * p[1].x;
    jx = cr;
    jy = ci;
    jz = 0.5 * ((p[0].x * p[0].x + p[0].y * p[0].y) - (p[1].x * p[1].x + p[1].y * p[1].y));
  } else {
    // Jx = (1/√2)·tridiag(1): √2 Re(ψ0*ψ1 + ψ1*ψ2); Jy: √2 Im(ψ0*ψ1 + ψ1*ψ2); Jz = |ψ0|² − |ψ2|²
    const double ar = p[0].x * p[1].x + p[0].y * p[1].y + p[1].x * p[2].x + p[1].y * p[2].y;
    const double ai = p[0].x * p[1].y - p[0].y * p[1].x + p[1].x * p[2].y - p[1].y * p[2].x;
    jx = kSqrt2 * ar;
    jy = kSqrt2 * ai;
    jz = (p[0].x * p[0].x + p[0].y * p[0].y) - (p[2].x * p[2].x + p[2].y * p[2].y);
  }
  out[3 * s + 0] = jx;
  out[3 * s + 1] = jy;
  out[3 * s + 2] = jz;
}

// Input validation: bit 1 = non-finite sweep/state value, bit 2 = ω_q ≠ 0 in column qcol (analytic spin-one).
__global__ void validate_kernel(int64_t n_sweep, const double* sweep, int P, int qcol, int64_t n_state,
                                const double* state, int* flag) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int bad = 0;
  if (i < n_sweep) {
    const double v = sweep[i];
    if (!isfinite(v)) bad |= 1;
    if (qcol >= 0 && (i % P) == qcol && v != 0.0) bad |= 2;
  }
  if (i < n_state && !isfinite(state[i])) bad |= 1;
  if (bad) atomicOr(flag, bad);
}

// ---- host launchers -------------------------------------------------------------------------------------------
template <int D> size_t scan_ws_bytes(int64_t batch, int64_t k_count) { return ScanLayout<D>(batch, k_count).total; }

size_t scan_workspace_bytes(int dim, int64_t batch, int64_t k_count) {
  return dim == 2 ? scan_ws_bytes<2>(batch, k_count) : scan_ws_bytes<3>(batch, k_count);
}

size_t aggregate_workspace_bytes(int dim, int64_t batch, int64_t k_count) {
  // same tiling; per-tile totals live in the agg region
  return scan_workspace_bytes(dim, batch, k_count);
}

template <int D, bool SCAN>
static cudaError_t run_scan(int64_t batch, int64_t k_count, const double* U, const double* psi0, double* states,
                            double* aggregate, void* ws, cudaStream_t s, int* launches) {
  ScanLayout<D> L(batch, k_count);
  char* w = static_cast<char*>(ws);
  ScanArgs a;
  a.batch = batch;
  a.k_count = k_count;
  a.tiles_per_sweep = L.tiles_per_sweep;
  a.U = reinterpret_cast<const double2*>(U);
  a.psi0 = reinterpret_cast<const double2*>(psi0);
  a.states = reinterpret_cast<double2*>(states);
  a.ticket = reinterpret_cast<unsigned long long*>(w);
  a.flags = reinterpret_cast<int*>(w + L.off_flags);
  a.agg = reinterpret_cast<double2*>(w + L.off_agg);
  a.psi_end = reinterpret_cast<double2*>(w + L.off_psi);
  a.aggregate_out = a.agg;
  cudaError_t e = cudaMemsetAsync(w, 0, L.off_agg, s);   // ticket + flags
  if (e != cudaSuccess) return e;
  if (L.ntiles > 0x7fffffffLL) return cudaErrorInvalidValue;
  constexpr int TILE = tile_size<D>();
  constexpr size_t smem = sizeof(double2) * (size_t)TILE * D * (D + (SCAN ? 1 : 0));
  static bool attr_set = false;
  if (!attr_set) {
    e = cudaFuncSetAttribute(scan_kernel<D, SCAN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  scan_kernel<D, SCAN><<<(unsigned)L.ntiles, kScanThreads, smem, s>>>(a);
  ++*launches;
  e = cudaGetLastError();
  if (e != cudaSuccess || SCAN) return e;
  combine_tiles_kernel<D><<<(unsigned)((batch + 127) / 128), 128, 0, s>>>(batch, L.tiles_per_sweep, a.agg,
                                                                          reinterpret_cast<double2*>(aggregate));
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_scan(int dim, int64_t batch, int64_t k_count, const double* U, const double* psi0, double* states,
                        void* ws, cudaStream_t s, int* launches) {
  return dim == 2 ? run_scan<2, true>(batch, k_count, U, psi0, states, nullptr, ws, s, launches)
                  : run_scan<3, true>(batch, k_count, U, psi0, states, nullptr, ws, s, launches);
}

cudaError_t launch_aggregate(int dim, int64_t batch, int64_t k_count, const double* U, double* aggregate, void* ws,
                             cudaStream_t s, int* launches) {
  return dim == 2 ? run_scan<2, false>(batch, k_count, U, nullptr, nullptr, aggregate, ws, s, launches)
                  : run_scan<3, false>(batch, k_count, U, nullptr, nullptr, aggregate, ws, s, launches);
}

cudaError_t launch_compose_carry(int dim, int64_t batch, int part, const double* aggs, const double* psi0,
                                 double* carry, cudaStream_t s) {
  const unsigned g = (unsigned)((batch + 127) / 128);
  if (dim == 2)
    compose_carry_kernel<2><<<g, 128, 0, s>>>(batch, part, reinterpret_cast<const double2*>(aggs),
                                              reinterpret_cast<const double2*>(psi0), reinterpret_cast<double2*>(carry));
  else
    compose_carry_kernel<3><<<g, 128, 0, s>>>(batch, part, reinterpret_cast<const double2*>(aggs),
                                              reinterpret_cast<const double2*>(psi0), reinterpret_cast<double2*>(carry));
  return cudaGetLastError();
}

cudaError_t launch_spin_projection(int dim, int64_t n, const double* states, double* out, cudaStream_t s) {
  const unsigned g = (unsigned)((n + 127) / 128);
  if (dim == 2) spin_projection_kernel<2><<<g, 128, 0, s>>>(n, reinterpret_cast<const double2*>(states), out);
  else spin_projection_kernel<3><<<g, 128, 0, s>>>(n, reinterpret_cast<const double2*>(states), out);
  return cudaGetLastError();
}

cudaError_t launch_validate(int64_t n_sweep, const double* sweep, int P, int qcol, int64_t n_state,
                            const double* state, int* flag, cudaStream_t s) {
  const int64_t n = n_sweep > n_state ? n_sweep : n_state;
  if (n <= 0) return cudaSuccess;
  validate_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n_sweep, sweep, P, qcol, n_state, state, flag);
  return cudaGetLastError();
}

}  // namespace ssb
