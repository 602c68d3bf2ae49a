// scan.cu — state propagation and the small kernels around it.
//
// ψ_{k+1} = U_k ψ_k (Eq. integration_compilation) is a linear recurrence; the paper runs it sequentially
// on the CPU.  Here it is an associative matrix-product scan (combine = later·earlier), with one kernel per
// problem shape (run_state_scan picks; DESIGN.md §5 "State propagation"):
//   * chain_kernel — batch ≥ 4096 (dense spin-one: 2304): one thread per sweep chains its states, operators
//     TMA-streamed through a per-sweep ring of bulk copies as deep as the shared memory allows;
//   * scan_coop_kernel — problems whose operators fit in L2: one cooperative wave, thread products, block
//     Kogge–Stone, one grid barrier, predecessor aggregates, states;
//   * run_chain_kernel — the fused path's states pass (the interval kernel wrote run products) and, in AGG mode, the
//     first pass of the standalone two-pass scan of compact operators: one lane per run of 4–32 operators, a warp's
//     32 runs staged by coalesced cp.async, states out with coalesced stores;
//   * scan3_kernel — dense long sweeps at moderate batch: persistent CTAs over tensor-TMA-staged tiles with
//     decoupled look-back (aggregate published, predecessors' aggregates multiplied until an inclusive prefix);
//   * scan2_kernel — the rest: double-buffered tiles, warp Kogge–Stone, block combine, warp-parallel look-back.
// HBM traffic per interval: read U_k + write ψ_{k+1} (2·dim doubles).  U_k travels either as the dense dim×dim complex
// matrix (the public layout: 144 / 64 B) or, for the SU(2)-form interval kernels (spin-half, analytic spin-one) when
// U_k is not an output, as the SU(2) element (a, b) (32 B) the kernel accumulates: 192 / 96 B per interval dense,
// 80 / 64 B compact.  Every scan is HBM bound.  The kernels are templated on the operator type M
// (CM<D> dense, SU<D> compact acting on dim-D states, ops.cuh), so each path exists for both formats.
#include <cooperative_groups.h>
#include <cuda/atomic>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>

#include <cuda.h>

#include "kernels.h"
#include "ops.cuh"

namespace ssb {

// Per-device host caches (function attributes, occupancy-derived grids, SM counts): cudaFuncSetAttribute applies to
// the current device's context, so every value is keyed by the device ordinal; atomics make concurrent first calls
// benign (both compute the same value).
constexpr int kMaxDevices = 64;
struct DeviceCache {
  std::atomic<int> v[kMaxDevices] = {};
  int get(int dev) const { return (dev >= 0 && dev < kMaxDevices) ? v[dev].load(std::memory_order_acquire) : 0; }
  void set(int dev, int x) { if (dev >= 0 && dev < kMaxDevices) v[dev].store(x, std::memory_order_release); }
};
static int device_sms(int dev) {
  static DeviceCache c;
  int n = c.get(dev);
  if (n == 0) {
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    c.set(dev, n);
  }
  return n;
}
static int current_device() {
  int dev = 0;
  return cudaGetDevice(&dev) == cudaSuccess ? dev : 0;
}

template <int D> struct ScanCfg;
template <> struct ScanCfg<2> { static constexpr int kItems = 4; };
template <> struct ScanCfg<3> { static constexpr int kItems = 2; };
constexpr int kScanThreads = 128;
template <int D> constexpr int tile_size() { return kScanThreads * ScanCfg<D>::kItems; }

enum { FLAG_EMPTY = 0, FLAG_AGG = 1, FLAG_PREFIX = 2 };

// Operator types (CM<D>, SU<D>), their products, loads, shuffles and ⟨J⟩: ops.cuh.

// Workspace layouts (all offsets 256-byte aligned): [ticket u64][flags int32 × ntiles][agg op × ntiles]
// [psi_end dim c128 × ntiles]; the v1 layout below also sizes the per-tile totals of ss_chain_aggregate.
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
  double2* aggregate_out;    // [ntiles][D][D] per-tile totals
};

// Per-tile aggregates for the time partition (ss_chain_aggregate): a block stages one tile of kTile consecutive
// operators of one sweep in shared memory, each thread multiplies its kItems consecutive operators, a warp shuffle
// tree and one pass over the warp totals give the tile total T = U_{last} ⋯ U_{first}; combine_tiles_kernel then
// multiplies the tiles of each sweep in order.  No look-back: the result is the same fixed association on every rank.
template <int D>
__global__ void __launch_bounds__(kScanThreads) aggregate_kernel(const ScanArgs a) {
  constexpr int C = ScanCfg<D>::kItems;
  constexpr int TILE = kScanThreads * C;
  constexpr int NW = kScanThreads / 32;
  extern __shared__ double2 smem[];          // [TILE·D·D] operators
  double2* sU = smem;
  __shared__ double2 sWarpTot[NW][D * D];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long ticket = blockIdx.x;
  const long long b = ticket / a.tiles_per_sweep;
  const long long j = ticket - b * a.tiles_per_sweep;
  const long long k0 = j * TILE;
  const int n_items = (int)min((long long)TILE, a.k_count - k0);
  const double2* gU = a.U + ((size_t)b * a.k_count + k0) * D * D;
  for (int e = tid; e < n_items * D * D; e += kScanThreads) sU[e] = __ldcs(gU + e);
  __syncthreads();
  CM<D> P;                                   // thread product U_{c+C−1} ⋯ U_c
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
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {   // warp total, later·earlier
    const CM<D> q = cm_shfl_down(P, off);
    if ((lane & (2 * off - 1)) == 0) P = cm_mul(q, P);
  }
  if (lane == 0) cm_store(sWarpTot[warp], P);
  __syncthreads();
  if (tid == 0) {
    CM<D> tot, t;
    cm_eye(tot);
    for (int w = 0; w < NW; ++w) { cm_load(sWarpTot[w], t); tot = cm_mul(t, tot); }
    cm_store(a.aggregate_out + (size_t)ticket * D * D, tot);
  }
}

// ---- state scan v2: persistent CTAs, TMA bulk-copy double buffering, j-major tiles, warp-parallel look-back ----
//
// Tile (b, j) covers intervals [j·TILE, (j+1)·TILE) of sweep b; tickets are j-major (ticket = j·batch + b), so the
// predecessor of a tile is ticket − batch: with many sweeps the predecessor has long finished and the look-back is a
// single flag read; with one sweep the look-back walks up to 32 predecessors per round in parallel (one lane each)
// and multiplies their aggregates with a shuffle tree.  Each CTA is persistent: while it computes tile t it has
// already issued the TMA bulk copy (cp.async.bulk → UBLKCP) of its next tile's operators into the other shared-
// memory stage, so HBM reads overlap the FP64 work.
#ifndef SS_SCAN2_NT
#define SS_SCAN2_NT 128
#endif
#ifndef SS_SCAN2_TILE3
#define SS_SCAN2_TILE3 512
#endif
#ifndef SS_SCAN2_TILE2
#define SS_SCAN2_TILE2 1024
#endif
// tile: 1024 intervals of dim-2 states, 512 of dim-3 (either operator format)
template <class M> struct Scan2Cfg {
  static constexpr int NT = SS_SCAN2_NT, C = (M::SD == 2 ? SS_SCAN2_TILE2 : SS_SCAN2_TILE3) / SS_SCAN2_NT;
};
template <class M> constexpr int scan2_tile() { return Scan2Cfg<M>::NT * Scan2Cfg<M>::C; }
// Per-thread shared-memory slots (a thread's C operators / C states), strides padded to an odd number of 16-byte
// words so the warp's LDS.128/STS.128 at equal offsets of 32 slots are bank-conflict free.
template <class M> __host__ __device__ constexpr int scan2_u_stride() { return (Scan2Cfg<M>::C * M::W) | 1; }
template <class M> __host__ __device__ constexpr int scan2_s_stride() { return (Scan2Cfg<M>::C * M::SD) | 1; }
template <class M> __host__ __device__ constexpr int scan2_j_stride() { return (Scan2Cfg<M>::C * 3) | 1; }  // doubles
template <class M> constexpr size_t scan2_smem() {
  return sizeof(double2) * (size_t)Scan2Cfg<M>::NT * (2 * scan2_u_stride<M>() + scan2_s_stride<M>()) +
         sizeof(double) * (size_t)Scan2Cfg<M>::NT * scan2_j_stride<M>() + 64;
}

template <class M> struct Scan2Layout {
  int64_t tiles_per_sweep, ntiles;
  size_t off_flags, off_agg, off_psi, total;
  Scan2Layout(int64_t batch, int64_t k_count) {
    tiles_per_sweep = (k_count + scan2_tile<M>() - 1) / scan2_tile<M>();
    ntiles = batch * tiles_per_sweep;
    off_flags = 256;
    off_agg = align256(off_flags + sizeof(int) * (size_t)ntiles);
    off_psi = align256(off_agg + sizeof(double2) * M::W * (size_t)ntiles);
    total = align256(off_psi + sizeof(double2) * M::SD * (size_t)ntiles);
  }
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst_smem, const void* src_gmem, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

struct Scan2Args {
  int64_t batch, k_count, tiles_per_sweep, ntiles;
  const double2* U;
  const double2* psi0;
  double2* states;   // or NULL
  double* spin;      // [batch][K+1][3] or NULL
  unsigned long long* ticket;
  int* flags;
  double2* agg;
  double2* psi_end;
};

template <class M>
__global__ void __launch_bounds__(Scan2Cfg<M>::NT) scan2_kernel(const Scan2Args a) {
  constexpr int D = M::SD, W = M::W;
  constexpr int NT = Scan2Cfg<M>::NT, C = Scan2Cfg<M>::C, TILE = NT * C, NW = NT / 32;
  constexpr int SU = scan2_u_stride<M>(), SS = scan2_s_stride<M>();
  extern __shared__ __align__(128) double2 smem2[];
  double2* sU[2] = {smem2, smem2 + NT * SU};                // [stage][thread][SU]
  double2* sPsi = smem2 + 2 * NT * SU;                      // [thread][SS]
  constexpr int SJ = scan2_j_stride<M>();
  double* sJ = reinterpret_cast<double*>(sPsi + NT * SS);   // [thread][SJ]
  __shared__ __align__(8) uint64_t sBar[2];
  __shared__ double2 sWarpTot[NW][W];
  __shared__ double2 sWarpPre[NW][W];
  __shared__ double2 sPsiIn[D];
  __shared__ long long sNext;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  auto tile_of = [&](long long t, long long& b, long long& j) { j = t / a.batch; b = t - j * a.batch; };
  // every thread bulk-copies its own C consecutive operators of tile t into its padded slot of `stage`
  auto issue = [&](long long t, int stage) {
    long long b, j;
    tile_of(t, b, j);
    const long long k0 = j * TILE + (long long)tid * C;
    const int n = (int)max(0LL, min((long long)C, a.k_count - k0));
    if (n > 0) {
      const unsigned bytes = (unsigned)(n * W * sizeof(double2));
      mbar_expect_tx(&sBar[stage], bytes);
      tma_load_1d(sU[stage] + tid * SU, a.U + ((size_t)b * a.k_count + k0) * W, bytes, &sBar[stage]);
    } else {
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&sBar[stage])) : "memory");
    }
  };

  if (tid == 0) {
    mbar_init(&sBar[0], NT);
    mbar_init(&sBar[1], NT);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    sNext = (long long)atomicAdd(a.ticket, 1ull);
  }
  __syncthreads();
  long long t = sNext;
  if (t < a.ntiles) issue(t, 0);
  unsigned phase[2] = {0u, 0u};
  int stage = 0;
  while (t < a.ntiles) {
    // Take the next ticket only now (one tile ahead, like every other CTA), so the tiles in flight at any moment
    // form a contiguous ticket range; then prefetch it into the other stage (consumed last iteration).
    __syncthreads();
    if (tid == 0) sNext = (long long)atomicAdd(a.ticket, 1ull);
    __syncthreads();
    const long long nx = sNext;
    if (nx < a.ntiles) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(nx, stage ^ 1);
    }
    long long b, j;
    tile_of(t, b, j);
    const long long k0 = j * TILE;
    const int n_items = (int)min((long long)TILE, a.k_count - k0);
    mbar_wait(&sBar[stage], phase[stage]);
    phase[stage] ^= 1u;
    const double2* U = sU[stage] + tid * SU;                // this thread's C operators

    // thread aggregate, warp inclusive scan, warp totals
    M P;
    cm_eye(P);
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const int it = tid * C + c;
      if (it < n_items) {
        M u;
        cm_load(U + c * W, u);
        P = cm_mul(u, P);
      }
    }
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const M q = cm_shfl_up(P, off);
      if (lane >= off) P = cm_mul(P, q);
    }
    M E = cm_shfl_up(P, 1);
    if (lane == 0) cm_eye(E);
    if (lane == 31) cm_store(sWarpTot[warp], P);
    __syncthreads();

    if (warp == 0) {
      // scan of the warp totals (lanes < NW), exclusive prefixes to shared memory, block total in lane NW−1
      M T;
      if (lane < NW) cm_load(sWarpTot[lane], T); else cm_eye(T);
#pragma unroll
      for (int off = 1; off < NW; off <<= 1) {
        const M q = cm_shfl_up(T, off);
        if (lane >= off) T = cm_mul(T, q);
      }
      M Wx = cm_shfl_up(T, 1);
      if (lane == 0) cm_eye(Wx);
      if (lane < NW) cm_store(sWarpPre[lane], Wx);
      // block total to every lane
      const M tot = cm_shfl_idx(T, NW - 1);
      cuda::atomic_ref<int, cuda::thread_scope_device> my_flag(a.flags[t]);
      double pr[D], pi[D];
      if (j == 0) {
#pragma unroll
        for (int d = 0; d < D; ++d) { const double2 v = a.psi0[b * D + d]; pr[d] = v.x; pi[d] = v.y; }
      } else {
        if (lane == 0) {
          cm_store(a.agg + (size_t)t * W, tot);
          my_flag.store(FLAG_AGG, cuda::memory_order_release);
        }
        // warp-parallel look-back: lane ℓ inspects predecessor j − 1 − ℓ − 32r
        M Mlb;
        cm_eye(Mlb);
        long long jb = j - 1;
        for (;;) {
          const long long jq = jb - lane;
          const long long q = jq * a.batch + b;
          int fv = FLAG_PREFIX;                       // lanes before tile 0 never matter (tile 0 is PREFIX)
          if (jq >= 0) {
            cuda::atomic_ref<int, cuda::thread_scope_device> f(a.flags[q]);
            while ((fv = f.load(cuda::memory_order_acquire)) == FLAG_EMPTY) __nanosleep(32);
          }
          const unsigned pm = __ballot_sync(0xffffffffu, fv == FLAG_PREFIX);
          const int first = pm ? __ffs(pm) - 1 : 32;
          if (first > 0) {                            // product of aggregates of lanes < first (nearest first)
            M A;
            if (lane < first) cm_load_cg(a.agg + (size_t)q * W, A); else cm_eye(A);
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
              const M o = cm_shfl_down(A, off);
              if ((lane & (2 * off - 1)) == 0) A = cm_mul(A, o);
            }
            Mlb = cm_mul(Mlb, A);                     // meaningful in lane 0
          }
          if (first < 32) {
            double er[D], ei[D];
            if (lane == first)
              for (int d = 0; d < D; ++d) { const double2 v = __ldcg(a.psi_end + q * D + d); er[d] = v.x; ei[d] = v.y; }
#pragma unroll
            for (int d = 0; d < D; ++d) {
              er[d] = __shfl_sync(0xffffffffu, er[d], first);
              ei[d] = __shfl_sync(0xffffffffu, ei[d], first);
            }
            cm_apply(Mlb, er, ei, pr, pi);            // valid in lane 0
            break;
          }
          jb -= 32;
        }
#pragma unroll
        for (int d = 0; d < D; ++d) {
          pr[d] = __shfl_sync(0xffffffffu, pr[d], 0);
          pi[d] = __shfl_sync(0xffffffffu, pi[d], 0);
        }
      }
      if (lane == 0) {
        double er[D], ei[D];
        cm_apply(tot, pr, pi, er, ei);
        for (int d = 0; d < D; ++d) a.psi_end[t * D + d] = make_double2(er[d], ei[d]);
        my_flag.store(FLAG_PREFIX, cuda::memory_order_release);
        for (int d = 0; d < D; ++d) sPsiIn[d] = make_double2(pr[d], pi[d]);
        if (j == 0) {
          if (a.states)
            for (int d = 0; d < D; ++d) a.states[(size_t)b * (a.k_count + 1) * D + d] = make_double2(pr[d], pi[d]);
          if (a.spin) {
            double jj3[3];
            spin_of<D>(pr, pi, jj3);
            for (int q = 0; q < 3; ++q) a.spin[(size_t)b * (a.k_count + 1) * 3 + q] = jj3[q];
          }
        }
      }
    }
    __syncthreads();

    // apply: ψ = (E·W_w)·ψ_in, then the thread's own operators
    M Wp;
    cm_load(sWarpPre[warp], Wp);
    const M X = cm_mul(E, Wp);
    double xr[D], xi[D], yr[D], yi[D];
#pragma unroll
    for (int d = 0; d < D; ++d) { xr[d] = sPsiIn[d].x; xi[d] = sPsiIn[d].y; }
    cm_apply(X, xr, xi, yr, yi);
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const int it = tid * C + c;
      if (it < n_items) {
        M u;
        cm_load(U + c * W, u);
        cm_apply(u, yr, yi, xr, xi);
#pragma unroll
        for (int d = 0; d < D; ++d) { yr[d] = xr[d]; yi[d] = xi[d]; sPsi[tid * SS + c * D + d] = make_double2(xr[d], xi[d]); }
        if (a.spin) {
          double jj3[3];
          spin_of<D>(xr, xi, jj3);
          for (int q = 0; q < 3; ++q) sJ[tid * SJ + c * 3 + q] = jj3[q];
        }
      }
    }
    __syncthreads();
    double2* gS = a.states + ((size_t)b * (a.k_count + 1) + k0 + 1) * D;
    if (a.states)
      for (int e = tid; e < n_items * D; e += NT) __stcs(gS + e, sPsi[(e / (C * D)) * SS + e % (C * D)]);
    if (a.spin) {
      double* gJ = a.spin + ((size_t)b * (a.k_count + 1) + k0 + 1) * 3;
      for (int e = tid; e < n_items * 3; e += NT) __stcs(gJ + e, sJ[(e / (C * 3)) * SJ + e % (C * 3)]);
    }
    t = nx;
    stage ^= 1;
  }
}

// ---- state scan v3 (small batches / long sweeps): thread-contiguous tiles, one look-back per tile -------------------
//
// Thread i of a tile owns the IPT = nst·C consecutive intervals [i·IPT, (i+1)·IPT) (nst stages of C; the tile is
// NT·IPT intervals, up to 4096 spin-one / 8192 spin-half).  Viewing one sweep's U as rows of IPT intervals, stage s of
// a tile is the box {C intervals of column s} × {NT rows}: ONE 4-D tensor-TMA load (padded by one out-of-bounds 16-B
// element per row so the per-thread slots land at an odd 16-B pitch — conflict-free).  Pass A streams the tile from
// HBM through an NSTAGE-deep full/empty mbarrier ring and folds each thread's operators into its running product P_i
// in registers — no block-level work per stage.  One warp Kogge–Stone + warp-total combine turns the P_i into
// exclusive prefixes X_i and the tile aggregate G; G is published and the decoupled look-back (warp 0, 32
// predecessors per round, j-major tickets) yields ψ_in.  Pass B re-streams the tile (L2-resident: 148 CTAs × ≤ 0.6 MB)
// and each thread propagates y = X_i ψ_in through its intervals; the states of a stage are staged in shared memory
// and leave as ONE tensor-TMA store.  The last tile of a sweep (when K is not a multiple of the tile) falls back to
// per-thread bulk copies.  The tile size nst adapts so that small problems still fill the GPU.
#ifndef SS_SCAN3_MAXST
#define SS_SCAN3_MAXST 16   // stages per pass in the largest tile
#endif
#ifndef SS_SCAN3_NSTAGE
#define SS_SCAN3_NSTAGE 5   // TMA ring depth; shallower rings fit 2 CTAs per SM (tuning knob)
#endif
// C intervals per thread and stage: ≈ 256 B of operators per row (dense: 4 × 64 B, 2 × 144 B); compact SU(2)
// operators (32 B) take C = 4 and a deeper ring (8 stages) so that as many bytes are in flight.
#ifndef SS_SCAN3_NT9
#define SS_SCAN3_NT9 128     // threads per CTA for dense spin-one operators (tuning knob)
#endif
#ifndef SS_SCAN3_NSTAGE9
#define SS_SCAN3_NSTAGE9 SS_SCAN3_NSTAGE
#endif
#ifndef SS_SCAN3_C9
#define SS_SCAN3_C9 0        // intervals per row and stage for dense spin-one operators (0: 256 / NT)
#endif
template <class M> struct Scan3Cfg {
  static constexpr int D = M::SD, W = M::W;
  static constexpr int NT = (W == 9) ? SS_SCAN3_NT9 : 128, NW = NT / 32;
  static constexpr int C = (W == 9) ? (SS_SCAN3_C9 > 0 ? SS_SCAN3_C9 : 256 / NT) : 4;
  static constexpr int NSTAGE = (W == 2) ? 8 : (W == 9 ? SS_SCAN3_NSTAGE9 : SS_SCAN3_NSTAGE), MAXST = SS_SCAN3_MAXST;
  static constexpr int SU = C * W + 1;       // slot pitch in double2: odd → conflict-free per-thread reads
  static constexpr int SS = C * D + 1;       // state staging pitch in double2
};
template <class M> constexpr size_t scan3_smem() {
  return sizeof(double2) * (size_t)Scan3Cfg<M>::NT * (Scan3Cfg<M>::NSTAGE * Scan3Cfg<M>::SU + 2 * Scan3Cfg<M>::SS);
}
template <class M> struct Scan3Layout {
  int64_t tile, tiles_per_sweep, ntiles;
  size_t off_flags, off_agg, off_psi, total;
  Scan3Layout(int64_t batch, int64_t k_count, int nst) {
    tile = (int64_t)Scan3Cfg<M>::NT * Scan3Cfg<M>::C * nst;
    tiles_per_sweep = (k_count + tile - 1) / tile;
    ntiles = batch * tiles_per_sweep;
    off_flags = 256;
    off_agg = align256(off_flags + sizeof(int) * (size_t)ntiles);
    off_psi = align256(off_agg + sizeof(double2) * M::W * (size_t)ntiles);
    total = align256(off_psi + sizeof(double2) * M::SD * (size_t)ntiles);
  }
};
struct Scan3Args {
  Scan2Args s;
  int nst;
  int tensor_u, tensor_s;   // tensor maps valid (some full tile exists / states requested)
};

__device__ __forceinline__ void bulk_store(void* dst_gmem, const void* src_smem, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst_gmem), "r"(smem_u32(src_smem)),
               "r"(bytes)
               : "memory");
}
#ifndef SS_SCAN3_HINTS
#define SS_SCAN3_HINTS 1   // L2 eviction hints: pass A evict_last (re-read by pass B), pass B + state stores evict_first
#endif
__device__ __forceinline__ void tma_load_4d(void* dst_smem, const CUtensorMap* tm, int c0, int c1, int c2, int c3,
                                            uint64_t* bar, uint64_t policy) {
#if SS_SCAN3_HINTS
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4, %5}], [%6], %7;"
      ::"r"(smem_u32(dst_smem)), "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
#else
  (void)policy;
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
      ::"r"(smem_u32(dst_smem)), "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
#endif
}
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* tm, const void* src_smem, int c0, int c1, int c2, int c3,
                                             uint64_t policy) {
#if SS_SCAN3_HINTS
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2, %3, %4}], [%5], %6;"
               ::"l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(src_smem)), "l"(policy)
               : "memory");
#else
  (void)policy;
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];"
               ::"l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(src_smem))
               : "memory");
#endif
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <class M>
__global__ void __launch_bounds__(Scan3Cfg<M>::NT, 1)
    scan3_kernel(const __grid_constant__ Scan3Args A3, const __grid_constant__ CUtensorMap tmU,
                 const __grid_constant__ CUtensorMap tmS) {
  constexpr int D = M::SD, W = M::W;
  constexpr int NT = Scan3Cfg<M>::NT, NW = Scan3Cfg<M>::NW, C = Scan3Cfg<M>::C, NSTAGE = Scan3Cfg<M>::NSTAGE;
  constexpr int SU = Scan3Cfg<M>::SU, SS = Scan3Cfg<M>::SS;
  const Scan2Args& a = A3.s;
  const int nst = A3.nst, IPT = nst * C, LPT = 2 * nst;   // stages per pass, intervals per thread, loads per tile
  const long long TILE = (long long)NT * IPT;
  extern __shared__ __align__(128) double2 smem5[];
  double2* const sStage = smem5 + NSTAGE * NT * SU;         // [2][NT][SS] state staging
  __shared__ __align__(8) uint64_t sFull[NSTAGE];
  __shared__ __align__(8) uint64_t sEmpty[NSTAGE];
  __shared__ double2 sWarpTot[NW][W];
  __shared__ double2 sPsiIn[D];
  __shared__ double2 sPsiEnd[D];
  __shared__ double2 sTot[W];
  __shared__ double2 sM[W];
  __shared__ double2 sWarpAgg[NW][W];
  __shared__ unsigned sBal[NW];
  __shared__ long long sNext;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  auto buf = [&](long long n) { return smem5 + (int)(n % NSTAGE) * NT * SU; };

  // The CTA's load sequence: per tile LPT loads, pass A stages 0..nst−1 then pass B stages 0..nst−1.  Only the current
  // tile and the next have known tickets, so the issue cursor `ic` (relative to the current tile's first load) stays
  // below 2·LPT.  Ring slots and mbarrier parities advance incrementally: no 64-bit division on the per-stage path.
  long long tcur = 0, tnext = 0, n_iss = 0;
  long long jc = 0, bc = 0, jn = 0, bn = 0;
  bool fc = false, fn = false;                               // current / next tile is full (tensor path)
  int ic = 0, cc = 0, ix = 0, cx = 0;
  unsigned iph = 0, cph = 0;
  uint64_t pol_keep = 0, pol_stream = 0;
#if SS_SCAN3_HINTS
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_keep));
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_stream));
#endif
  auto issue = [&](int r_rel) {
    const bool sel = r_rel >= LPT;
    const int r = sel ? r_rel - LPT : r_rel;
    const bool passB = r >= nst;
    const int s = passB ? r - nst : r;
    const long long j = sel ? jn : jc, b = sel ? bn : bc;
    const int x = ix;
    if (sel ? fn : fc) {                                     // full tile: one tensor load by thread 0
      if (tid == 0) {
        if (n_iss >= NSTAGE) mbar_wait(&sEmpty[x], iph ^ 1u);
        mbar_expect_tx(&sFull[x], (unsigned)(NT * SU * sizeof(double2)));
        tma_load_4d(smem5 + x * NT * SU, &tmU, 0, s, (int)(j * NT), (int)b, &sFull[x], passB ? pol_stream : pol_keep);
      } else {
        mbar_arrive(&sFull[x]);
      }
    } else {
      // last tile of a sweep (K not a multiple of the tile): every thread copies its own ≤ C operators with 16-byte
      // cp.async, all threads at once, and the mbarrier counts its arrival when they land (arrive.noinc).  (Per-thread
      // bulk copies serialised their 128 issues through an elect loop: 1/3 of the tiles at K = 1e4.)
      const long long k0 = j * TILE + (long long)tid * IPT + (long long)s * C;
      const int nit = (int)max(0LL, min((long long)C, a.k_count - k0));
      if (nit > 0) {
        const double2* src = a.U + ((size_t)b * a.k_count + k0) * W;
        double2* dst = smem5 + (x * NT + tid) * SU;
        for (int q = 0; q < nit * W; ++q)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst + q)), "l"(src + q) : "memory");
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&sFull[x])) : "memory");
      } else {
        mbar_arrive(&sFull[x]);
      }
    }
    ++n_iss;
    if (++ix == NSTAGE) { ix = 0; iph ^= 1u; }
  };
  auto top_up = [&]() {                                      // keep NSTAGE − 1 loads ahead of the consumer
    int lim = cc + NSTAGE - 1;
    const int known = (tnext < a.ntiles ? 2 : 1) * LPT;
    if (lim > known) lim = known;
    for (; ic < lim; ++ic) issue(ic);
  };
  auto consume = [&]() -> const double2* {
    mbar_wait(&sFull[cx], cph);
    return smem5 + (cx * NT + tid) * SU;
  };
  auto release = [&]() {                                     // this thread is done reading the current slot
    mbar_arrive(&sEmpty[cx]);
    if (++cx == NSTAGE) { cx = 0; cph ^= 1u; }
    ++cc;
  };

  if (tid == 0) {
    for (int i = 0; i < NSTAGE; ++i) {
      mbar_init(&sFull[i], NT);
      mbar_init(&sEmpty[i], NT);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (A3.tensor_u) asm volatile("prefetch.tensormap [%0];" ::"l"(&tmU) : "memory");
    if (A3.tensor_s) asm volatile("prefetch.tensormap [%0];" ::"l"(&tmS) : "memory");
    sNext = (long long)atomicAdd(a.ticket, 1ull);
  }
  __syncthreads();
  tcur = sNext;
  tnext = a.ntiles;
  jc = tcur / a.batch;
  bc = tcur - jc * a.batch;
  fc = (jc + 1) * TILE <= a.k_count;
  long long m = 0;                                           // pass-B stages done (staging buffer parity)
  while (tcur < a.ntiles) {
    __syncthreads();                                         // everyone has read sNext
    if (tid == 0) sNext = (long long)atomicAdd(a.ticket, 1ull);
    __syncthreads();
    tnext = sNext;
    jn = tnext / a.batch;
    bn = tnext - jn * a.batch;
    fn = (jn + 1) * TILE <= a.k_count;
    top_up();
    const long long j = jc, b = bc;
    const long long kt = j * TILE + (long long)tid * IPT;     // this thread's first interval
    const bool full = fc;
    // ---- pass A: P_i = U_{last} ⋯ U_{first} over this thread's intervals (HBM stream)
    M P;
    cm_eye(P);
    for (int s = 0; s < nst; ++s) {
      const double2* U = consume();
      const long long k0 = kt + (long long)s * C;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        if (k0 + c < a.k_count) {
          M u;
          cm_load(U + c * W, u);
          P = cm_mul(u, P);
        }
      }
      release();
      top_up();
    }
    // ---- block exclusive scan of the P_i: X_i = (P_{i-1} ⋯ P_0); tile aggregate G
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const M o = cm_shfl_up(P, off);
      if (lane >= off) P = cm_mul(P, o);
    }
    M X = cm_shfl_up(P, 1);
    if (lane == 0) cm_eye(X);
    if (lane == 31) cm_store(sWarpTot[warp], P);
    __syncthreads();
    {
      M Wpre, T;
      cm_eye(Wpre);
      for (int w = 0; w < warp; ++w) { cm_load(sWarpTot[w], T); Wpre = cm_mul(T, Wpre); }
      X = cm_mul(X, Wpre);
    }
    // ---- publish AGG, then a block-wide decoupled look-back: 128 predecessors per round (one round covers a wave)
    if (tid == 0) {
      M tot, T;
      cm_eye(tot);
      for (int w = 0; w < NW; ++w) { cm_load(sWarpTot[w], T); tot = cm_mul(T, tot); }
      cm_store(sTot, tot);
      if (j > 0) {
        cm_store(a.agg + (size_t)tcur * W, tot);
        cuda::atomic_ref<int, cuda::thread_scope_device>(a.flags[tcur]).store(FLAG_AGG, cuda::memory_order_release);
        cm_store(sM, [] { M e; cm_eye(e); return e; }());
      } else {
        for (int d = 0; d < D; ++d) sPsiIn[d] = a.psi0[b * D + d];
      }
    }
    if (j > 0) {
      for (long long jb = j - 1;; jb -= NT) {
        const long long jq = jb - tid;
        const long long tq = jq * a.batch + b;
        int fv = FLAG_PREFIX;                                  // jq < 0 is never reached: tile 0 publishes PREFIX
        if (jq >= 0) {
          cuda::atomic_ref<int, cuda::thread_scope_device> f(a.flags[tq]);
          while ((fv = f.load(cuda::memory_order_acquire)) == FLAG_EMPTY) __nanosleep(32);
        }
        const unsigned pm = __ballot_sync(0xffffffffu, fv == FLAG_PREFIX);
        if (lane == 0) sBal[warp] = pm;
        __syncthreads();
        int first = NT;
        for (int w = NW - 1; w >= 0; --w)
          if (sBal[w]) first = w * 32 + __ffs(sBal[w]) - 1;
        if (first > 0) {                                       // product of the AGGs before the first PREFIX
          M Ag;
          if (tid < first) cm_load_cg(a.agg + (size_t)tq * W, Ag); else cm_eye(Ag);
#pragma unroll
          for (int off = 1; off < 32; off <<= 1) {
            const M o = cm_shfl_down(Ag, off);
            if ((lane & (2 * off - 1)) == 0) Ag = cm_mul(Ag, o);
          }
          if (lane == 0) cm_store(sWarpAgg[warp], Ag);
        }
        if (tid == first) for (int d = 0; d < D; ++d) sPsiEnd[d] = __ldcg(a.psi_end + tq * D + d);
        __syncthreads();
        if (tid == 0) {
          M Mlb, T;
          cm_load(sM, Mlb);
          if (first > 0)
            for (int w = 0; w < NW; ++w) { cm_load(sWarpAgg[w], T); Mlb = cm_mul(Mlb, T); }
          if (first < NT) {
            double er[D], ei[D], pr[D], pi[D];
            for (int d = 0; d < D; ++d) { er[d] = sPsiEnd[d].x; ei[d] = sPsiEnd[d].y; }
            cm_apply(Mlb, er, ei, pr, pi);
            for (int d = 0; d < D; ++d) sPsiIn[d] = make_double2(pr[d], pi[d]);
          } else {
            cm_store(sM, Mlb);
          }
        }
        if (first < NT) break;
      }
    }
    if (tid == 0) {                                            // publish PREFIX: ψ at the end of this tile
      M tot;
      cm_load(sTot, tot);
      double pr[D], pi[D], er[D], ei[D];
      for (int d = 0; d < D; ++d) { pr[d] = sPsiIn[d].x; pi[d] = sPsiIn[d].y; }
      cm_apply(tot, pr, pi, er, ei);
      for (int d = 0; d < D; ++d) a.psi_end[tcur * D + d] = make_double2(er[d], ei[d]);
      cuda::atomic_ref<int, cuda::thread_scope_device>(a.flags[tcur]).store(FLAG_PREFIX, cuda::memory_order_release);
      if (j == 0) {
        if (a.states)
          for (int d = 0; d < D; ++d) a.states[(size_t)b * (a.k_count + 1) * D + d] = make_double2(pr[d], pi[d]);
        if (a.spin) {
          double jj3[3];
          spin_of<D>(pr, pi, jj3);
          for (int c = 0; c < 3; ++c) a.spin[(size_t)b * (a.k_count + 1) * 3 + c] = jj3[c];
        }
      }
    }
    __syncthreads();
    // ---- pass B: y = X_i ψ_in through this thread's intervals (L2 re-stream); states leave by TMA stores
    double yr[D], yi[D];
    {
      double xr[D], xi[D];
#pragma unroll
      for (int d = 0; d < D; ++d) { xr[d] = sPsiIn[d].x; xi[d] = sPsiIn[d].y; }
      cm_apply(X, xr, xi, yr, yi);
    }
    for (int s = 0; s < nst; ++s, ++m) {
      const double2* U = consume();
      double2* const st = sStage + ((int)(m & 1) * NT + tid) * SS;
      const long long k0 = kt + (long long)s * C;
      const int nit = (int)max(0LL, min((long long)C, a.k_count - k0));
#pragma unroll
      for (int c = 0; c < C; ++c) {
        if (c < nit) {
          M u;
          cm_load(U + c * W, u);
          double zr[D], zi[D];
          cm_apply(u, yr, yi, zr, zi);
#pragma unroll
          for (int d = 0; d < D; ++d) { yr[d] = zr[d]; yi[d] = zi[d]; st[c * D + d] = make_double2(zr[d], zi[d]); }
          if (a.spin) {
            double jj3[3];
            spin_of<D>(zr, zi, jj3);
            double* gJ = a.spin + ((size_t)b * (a.k_count + 1) + k0 + c + 1) * 3;
            for (int e = 0; e < 3; ++e) __stcs(gJ + e, jj3[e]);
          }
        }
      }
      release();
      if (a.states) {                                        // per warp: its 32 rows leave as one TMA store
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // staging writes → TMA store
        bulk_wait_read0();                                   // the store that read the other staging buffer is done
        __syncwarp();
        if (full) {
          if (lane == 0) {
            tma_store_4d(&tmS, sStage + ((int)(m & 1) * NT + warp * 32) * SS, 0, s, (int)(j * NT) + warp * 32, (int)b,
                         pol_stream);
            bulk_commit();
          }
        } else if (nit > 0) {                                // last tile: plain per-thread stores (no elect loop)
          double2* dstS = a.states + ((size_t)b * (a.k_count + 1) + k0 + 1) * D;
          for (int q = 0; q < nit * D; ++q) __stcs(dstS + q, st[q]);
        }
      }
      top_up();
    }
    tcur = tnext;
    jc = jn;
    bc = bn;
    fc = fn;
    ic -= LPT;
    cc -= LPT;
  }
  bulk_wait_all();
}

// ---- small problems: one cooperative wave with two grid-wide barriers instead of look-back -------------------------
//
// For problems whose operators fit in L2 (B·K·dim²·16 B ≤ 64 MB) and with few sweeps (C1, C2, C4's 1e6-interval
// sweep), the tile scan's decoupled look-back is latency-bound: every tile of one sweep runs in the same wave, so the
// last tile multiplies ~all predecessor aggregates (C2: 30 µs for 19 MB).  Here each sweep gets `cps` CTAs, CTA c owns
// a contiguous interval range and thread i of it a contiguous sub-range:
//   1. P_i = product of thread i's operators (HBM → L2), block Kogge–Stone → exclusive prefixes X_i, CTA aggregate G_c;
//   2. grid barrier; every CTA multiplies the ≤ cps − 1 aggregates of its sweep's predecessors (128 per round, one
//      ordered tree per round) into ψ_in = G_{c−1} ⋯ G_{first} ψ0;
//   3. y = X_i ψ_in, then thread i re-reads its operators (L2) and writes its states.
// All CTAs are co-resident (cooperative launch), so the barrier cannot deadlock.
struct CoopArgs {
  int64_t batch, k_count;
  int cps;                 // CTAs per sweep
  const double2* U;
  const double2* psi0;
  double2* states;         // or NULL
  double* spin;            // or NULL
  double2* agg;            // [grid][D·D] CTA aggregates (workspace)
};

// STAGED (one CTA per SM, the CTA's operators ≤ SS_COOP_STAGE_MAX bytes): the CTA's contiguous run of operators is
// brought into shared memory by ONE bulk copy (cp.async.bulk, mbarrier completion) before pass 1, so the whole run is
// in flight at once instead of each thread's dependent chain of 144-B loads (C2: 21 µs, long-scoreboard bound), and
// pass 3 re-reads it from shared memory instead of L2.
template <class M, bool STAGED>
__global__ void __launch_bounds__(128) scan_coop_kernel(const CoopArgs a) {
  namespace cg = cooperative_groups;
  constexpr int D = M::SD, W = M::W;
  constexpr int NT = 128, NW = NT / 32;
  __shared__ double2 sWarpTot[NW][W];
  __shared__ double2 sPsiIn[D];
  __shared__ double2 sM[W];
  __shared__ __align__(8) uint64_t sBar;
  extern __shared__ __align__(128) double2 sRun[];
  const int c = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t K = a.k_count;
  const int64_t b = c / a.cps;
  const int part = c - (int)b * a.cps;
  const bool has = b < a.batch;
  const int64_t per = (K + a.cps - 1) / a.cps;
  const int64_t k0 = has ? min((int64_t)part * per, K) : 0, k1 = has ? min(k0 + per, K) : 0;
  const int64_t m = (k1 - k0 + NT - 1) / NT;
  const int64_t t0 = min(k0 + (int64_t)tid * m, k1), t1 = min(t0 + m, k1);
  const double2* gU = a.U + (size_t)(has ? b : 0) * K * W;
  if constexpr (STAGED) {
    const unsigned bytes = (unsigned)((k1 - k0) * W * sizeof(double2));
    if (bytes > 0) {
      if (tid == 0) {
        mbar_init(&sBar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      }
      __syncthreads();
      if (tid == 0) {
        mbar_expect_tx(&sBar, bytes);
        tma_load_1d(sRun, gU + (size_t)k0 * W, bytes, &sBar);
      }
      mbar_wait(&sBar, 0);
    }
    gU = sRun - (size_t)k0 * W;                          // operator k at gU + k·W (shared memory)
  }
  // 1. thread product and block exclusive scan
  M P;
  cm_eye(P);
  // unrolled so several operators' loads are in flight per thread (the products are a dependent chain)
#pragma unroll 4
  for (int64_t k = t0; k < t1; ++k) {
    M u;
    cm_load(gU + (size_t)k * W, u);
    P = cm_mul(u, P);
  }
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const M o = cm_shfl_up(P, off);
    if (lane >= off) P = cm_mul(P, o);
  }
  M X = cm_shfl_up(P, 1);
  if (lane == 0) cm_eye(X);
  if (lane == 31) cm_store(sWarpTot[warp], P);
  __syncthreads();
  {
    M Wpre, T;
    cm_eye(Wpre);
    for (int w = 0; w < warp; ++w) { cm_load(sWarpTot[w], T); Wpre = cm_mul(T, Wpre); }
    X = cm_mul(X, Wpre);
    if (tid == 0) {
      M tot;
      cm_eye(tot);
      for (int w = 0; w < NW; ++w) { cm_load(sWarpTot[w], T); tot = cm_mul(T, tot); }
      cm_store(a.agg + (size_t)c * W, tot);
      cm_eye(tot);
      cm_store(sM, tot);
    }
  }
  cg::this_grid().sync();
  // 2. ψ_in: ordered product of the predecessors' aggregates (latest first), NT per round
  for (int q0 = part - 1; q0 >= 0; q0 -= NT) {
    const int q = q0 - tid;                                  // thread t holds G_{q0 − t} (later on the left)
    M Ag;
    if (q >= 0) cm_load_cg(a.agg + (size_t)(c - part + q) * W, Ag); else cm_eye(Ag);
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const M o = cm_shfl_down(Ag, off);
      if ((lane & (2 * off - 1)) == 0) Ag = cm_mul(Ag, o);
    }
    __syncthreads();                                         // sWarpTot reuse
    if (lane == 0) cm_store(sWarpTot[warp], Ag);
    __syncthreads();
    if (tid == 0) {
      M Mlb, T;
      cm_load(sM, Mlb);
      for (int w = 0; w < NW; ++w) { cm_load(sWarpTot[w], T); Mlb = cm_mul(Mlb, T); }
      cm_store(sM, Mlb);
    }
  }
  __syncthreads();
  if (tid == 0 && has) {
    M Mlb;
    cm_load(sM, Mlb);
    double xr[D], xi[D], yr[D], yi[D];
    for (int d = 0; d < D; ++d) { xr[d] = a.psi0[b * D + d].x; xi[d] = a.psi0[b * D + d].y; }
    cm_apply(Mlb, xr, xi, yr, yi);
    for (int d = 0; d < D; ++d) sPsiIn[d] = make_double2(yr[d], yi[d]);
    if (part == 0) {
      if (a.states)
        for (int d = 0; d < D; ++d) a.states[(size_t)b * (K + 1) * D + d] = make_double2(xr[d], xi[d]);
      if (a.spin) {
        double jj3[3];
        spin_of<D>(xr, xi, jj3);
        for (int e = 0; e < 3; ++e) a.spin[(size_t)b * (K + 1) * 3 + e] = jj3[e];
      }
    }
  }
  __syncthreads();
  if (!has) return;
  // 3. states of this thread's intervals
  double yr[D], yi[D];
  {
    double xr[D], xi[D];
#pragma unroll
    for (int d = 0; d < D; ++d) { xr[d] = sPsiIn[d].x; xi[d] = sPsiIn[d].y; }
    cm_apply(X, xr, xi, yr, yi);
  }
  double2* gS = a.states ? a.states + (size_t)b * (K + 1) * D : nullptr;
  double* gJ = a.spin ? a.spin + (size_t)b * (K + 1) * 3 : nullptr;
#pragma unroll 4
  for (int64_t k = t0; k < t1; ++k) {
    M u;
    cm_load(gU + (size_t)k * W, u);
    double zr[D], zi[D];
    cm_apply(u, yr, yi, zr, zi);
#pragma unroll
    for (int d = 0; d < D; ++d) { yr[d] = zr[d]; yi[d] = zi[d]; }
    if (gS)
#pragma unroll
      for (int d = 0; d < D; ++d) __stcs(gS + (k + 1) * D + d, make_double2(zr[d], zi[d]));
    if (gJ) {
      double jj3[3];
      spin_of<D>(zr, zi, jj3);
      for (int e = 0; e < 3; ++e) __stcs(gJ + (k + 1) * 3 + e, jj3[e]);
    }
  }
}

// ---- state chain for large batches: one thread per sweep, TMA-streamed ------------------------------------------
//
// With enough sweeps the sweeps alone give the parallelism to saturate HBM, so each thread runs its own sweep's
// recurrence ψ_{k+1} = U_k ψ_k sequentially (36 FP64 ops per interval, no matrix products, no look-back): the thread
// streams its sweep's operators through its own NST-stage ring of shared-memory slots, CH operators per bulk copy
// (cp.async.bulk → UBLKCP, one mbarrier per warp and stage), so NST − 1 copies per sweep are in flight while it
// applies the current CH.  One CTA per SM holds spc = ⌈batch / #SMs⌉ sweeps, dealt round-robin over its four warps
// (one per SM sub-partition: the recurrence is latency-bound per sweep, ≈ 300 cycles per interval, so four short
// warps beat one full one); the ring depth is what the shared memory gives spc slots (8192 sweeps: 56 slots × 2
// stages; 4096 sweeps, one GPU's shard of C3 at 2 GPUs: 28 × 4), so every SM keeps ≈ 100 KB of operator reads in
// flight.
constexpr int kChainThreads = 128;   // four warps
constexpr int kChainMaxSpc = 64;     // sweeps per CTA
#ifndef SS_COOP_MAXCPS
#define SS_COOP_MAXCPS 128     // CTAs per sweep of the cooperative scan (one predecessor round)
#endif
constexpr int64_t kChainMinBatch = 4096;
// Dense spin-one operators take the chain from 2304 sweeps: one sweep's serial recurrence costs ≈ 250 cycles per
// interval whatever the batch below ~3000 sweeps (1e4 intervals: 1.21 / 1.32 ms at 1024 / 2048 sweeps), while scan3
// runs at ≈ 0.46 of HBM, i.e. in time ∝ B (0.67 / 1.28 ms; profiles/r02/s42_scan3/scan_paths.txt): the crossover is
// near 2100 sweeps.  Other operators keep 4096 (compact ones prefer the two-pass scan).
template <class M> constexpr int64_t chain_min_batch_of() { return M::W == 9 ? 2304 : kChainMinBatch; }
#ifndef SS_CHAIN_CH
#define SS_CHAIN_CH 12   // operators per bulk copy: 4 / 8 / 12 → 2.9 / 5.2 / 5.4 TB/s on C3 (two stages)
#endif
#ifndef SS_CHAIN_MAX_STAGES
#define SS_CHAIN_MAX_STAGES 16
#endif
constexpr int kChainMaxStages = SS_CHAIN_MAX_STAGES;
constexpr int kChainSmemBudget = 220 * 1024;   // dynamic shared memory of the ring (one CTA per SM)
// compact SU(2) operators (32 B) are copied 48 at a time: ≈ 1.5 KB per copy like 12 dense spin-one operators
template <class M> struct ChainCfg { static constexpr int CH = M::W == 2 ? 4 * SS_CHAIN_CH : SS_CHAIN_CH; };
// Ring depth for spc lanes: the most stages (≤ kChainMaxStages) whose per-lane slots fit the budget, at least 2.
template <class M> __host__ __device__ constexpr int chain_slot_stride(int nst) {
  // stride padded to an odd number of 16-byte words so the lanes' LDS.128 at the same offset hit distinct banks (an
  // unpadded stride is a multiple of 128 B: a 32-way conflict)
  return (nst * ChainCfg<M>::CH * M::W) | 1;
}
template <class M> static int chain_stages(int spc) {
  int nst = kChainMaxStages;
  while (nst > 2 && (size_t)spc * chain_slot_stride<M>(nst) * sizeof(double2) > (size_t)kChainSmemBudget) --nst;
  return nst;
}

struct ChainArgs {
  int64_t batch, k_count;
  const double2* U;
  const double2* psi0;
  double2* states;   // [batch][K+1][D] or NULL
  double* spin;      // [batch][K+1][3] or NULL (⟨J⟩ fused into the write-out)
  int spc;           // sweeps per CTA (≤ kChainMaxSpc): spreads the batch over every SM
  int nst;           // ring stages per lane (2 … kChainMaxStages)
};

template <class M>
__global__ void __launch_bounds__(kChainThreads) chain_kernel(const ChainArgs a) {
  constexpr int D = M::SD, W = M::W;
  constexpr int CH = ChainCfg<M>::CH;
  extern __shared__ __align__(128) double2 smem3[];
  __shared__ __align__(8) uint64_t sBar[kChainThreads / 32][kChainMaxStages];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NST = a.nst;
  // this thread's sweep slot: the spc slots split into four contiguous runs, one per warp (adjacent lanes, adjacent
  // slots: the odd slot stride keeps their LDS.128 conflict-free)
  const int per_warp = (a.spc + 3) / 4;
  const int j = warp * per_warp + lane;
  const int64_t b = (int64_t)blockIdx.x * a.spc + j;
  const bool valid = lane < per_warp && j < a.spc && b < a.batch;
  // threads past spc own no slot (the CTA's shared memory holds spc slots) and only arrive on their warp's barriers
  double2* slot = smem3 + (size_t)(valid ? j : 0) * chain_slot_stride<M>(NST);
  if (lane == 0) {
    for (int st = 0; st < NST; ++st) mbar_init(&sBar[warp][st], 32);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const int64_t nchunks = (a.k_count + CH - 1) / CH;
  const double2* gU = a.U + (size_t)(valid ? b : 0) * a.k_count * W;
  auto issue = [&](int64_t c, int st) {
    const int64_t k0 = c * CH;
    const int n = valid ? (int)min((int64_t)CH, a.k_count - k0) : 0;
    const unsigned bytes = (unsigned)(n * W * sizeof(double2));
    if (bytes) {
      mbar_expect_tx(&sBar[warp][st], bytes);
      tma_load_1d(slot + st * (CH * W), gU + (size_t)k0 * W, bytes, &sBar[warp][st]);
    } else {
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&sBar[warp][st])) : "memory");
    }
  };
  for (int st = 0; st < NST && st < nchunks; ++st) issue(st, st);   // fill the ring
  double pr[D], pi[D];
  double2* gS = a.states ? a.states + (size_t)(valid ? b : 0) * (a.k_count + 1) * D : nullptr;
  double* gJ = a.spin ? a.spin + (size_t)(valid ? b : 0) * (a.k_count + 1) * 3 : nullptr;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const double2 v = valid ? a.psi0[b * D + d] : make_double2(0.0, 0.0);
    pr[d] = v.x; pi[d] = v.y;
    if (valid && gS) __stcs(gS + d, v);
  }
  if (valid && gJ) {
    double j[3];
    spin_of<D>(pr, pi, j);
    for (int q = 0; q < 3; ++q) __stcs(gJ + q, j[q]);
  }
  int st = 0;
  unsigned parity = 0u;   // phase parity of stage st's current use: flips each time the ring wraps
  for (int64_t c = 0; c < nchunks; ++c) {
    mbar_wait(&sBar[warp][st], parity);
    if (valid) {
      const int n = (int)min((int64_t)CH, a.k_count - c * CH);
      const double2* u = slot + st * (CH * W);
      const size_t kout = (size_t)(c * CH + 1);
      auto one = [&](int i) {
        double yr[D], yi[D];
        M m;
        cm_load(u + i * W, m);
        cm_apply(m, pr, pi, yr, yi);
#pragma unroll
        for (int d = 0; d < D; ++d) { pr[d] = yr[d]; pi[d] = yi[d]; }
        if (gS)
#pragma unroll
          for (int d = 0; d < D; ++d) __stcs(gS + (kout + i) * D + d, make_double2(yr[d], yi[d]));
        if (gJ) {
          double jj[3];
          spin_of<D>(pr, pi, jj);
          for (int q = 0; q < 3; ++q) __stcs(gJ + (kout + i) * 3 + q, jj[q]);
        }
      };
      if (n == CH) {   // full chunk unrolled: the operator loads are independent of ψ and issue ahead of the chain
#pragma unroll
        for (int i = 0; i < CH; ++i) one(i);
      } else {
        for (int i = 0; i < n; ++i) one(i);
      }
    }
    if (c + NST < nchunks) {   // refill the stage just consumed (generic reads before the async-proxy write)
      __syncwarp();
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(c + NST, st);
    }
    if (++st == NST) { st = 0; parity ^= 1u; }
  }
}

template <class M>
static cudaError_t run_chain(int64_t batch, int64_t k_count, const double* U, const double* psi0, double* states,
                             double* spin, cudaStream_t s, int* launches) {
  static DeviceCache attr;   // per device: the shared-memory opt-in applies to the current device's context
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (!attr.get(dev)) {
    e = cudaFuncSetAttribute(chain_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, kChainSmemBudget);
    if (e != cudaSuccess) return e;
    attr.set(dev, 1);
  }
  // Sweeps per CTA: at most kChainMaxSpc, and few enough that the CTAs cover every SM (8192 sweeps: 56 per CTA on
  // 147 CTAs instead of 64 on 128 — the per-SM TMA/L1 path, not HBM, limited the 128-CTA launch).
  const int sms = device_sms(dev);
  int spc = (int)std::min<int64_t>(kChainMaxSpc, (batch + sms - 1) / sms);
  if (spc < 1) spc = 1;
  const int nst = chain_stages<M>(spc);
  const size_t smem = (size_t)spc * chain_slot_stride<M>(nst) * sizeof(double2);
  ChainArgs a{batch, k_count, reinterpret_cast<const double2*>(U), reinterpret_cast<const double2*>(psi0),
              reinterpret_cast<double2*>(states), spin, spc, nst};
  chain_kernel<M><<<(unsigned)((batch + spc - 1) / spc), kChainThreads, smem, s>>>(a);
  ++*launches;
  return cudaGetLastError();
}

// ---- run chain of the fused path: one lane per run of SEG intervals, a warp per 32 consecutive runs ----------------
//
// The fused path picks SEG | K, so run g of the flat [batch][K] operator array covers operators [g·SEG, (g+1)·SEG)
// and a warp's 32 runs are ONE contiguous range of 32·SEG operators: the warp copies it into shared memory with
// coalesced 16-byte cp.async (LDGSTS, all in flight at once, no registers held), each run landing in its own slot at
// an odd 16-byte pitch (conflict-free per-lane reads).  Every lane then applies its run's operators from its start
// state phi[b][r] (the coarse scan's), writing state i over the slot's front while the operators sit at its back
// (state i never reaches an operator not yet read), and the warp streams each run's SEG contiguous states out with
// coalesced stores.  One-warp CTAs: the shared-memory footprint sets how many are resident per SM, each with its
// whole range in flight.
struct RunChainArgs {
  int64_t batch, k_count, nseg;   // nseg = K / SEG runs per sweep
  const double2* U;
  const double2* phi;             // [batch][nseg + 1][D]
  double2* states;                // [batch][K+1][D] or NULL
  double* spin;                   // [batch][K+1][3] or NULL
  double2* agg;                   // AGG mode: [batch][nseg] run products (W double2 each)
};
template <class M> __host__ __device__ constexpr int run_width() { return M::W > M::SD ? M::W : M::SD; }   // double2 per interval slot
template <class M, int SEG> __host__ __device__ constexpr int run_slot_stride() { return (SEG * run_width<M>()) | 1; }
template <class M, int SEG> constexpr size_t run_chain_smem() {
  return sizeof(double2) * 32 * (size_t)run_slot_stride<M, SEG>();
}

// AGG = true: the same staging, but each lane writes its run's product G = U_last ⋯ U_first (the reduce pass of the
// standalone two-pass scan, run_two_pass) instead of chaining states.
template <class M, int SEG, bool AGG = false>
__global__ void __launch_bounds__(32) run_chain_kernel(const RunChainArgs a) {
  constexpr int D = M::SD, W = M::W, STR = run_slot_stride<M, SEG>();
  constexpr int OFF = SEG * (run_width<M>() - W);            // operators at the back of the slot
  extern __shared__ __align__(128) double2 smem_rc[];
  const int lane = threadIdx.x;
  const int64_t nruns = a.batch * a.nseg;
  const int64_t g0 = (int64_t)blockIdx.x * 32;
  const int nw = (int)min((int64_t)32, nruns - g0);          // runs of this warp
  const double2* src = a.U + (size_t)g0 * SEG * W;
  const int nchunks = nw * SEG * W;                          // 16-byte chunks of the warp's range
#pragma unroll 4
  for (int c = lane; c < nchunks; c += 32) {
    const int j = c / (SEG * W), o = c - j * (SEG * W);     // run j of the warp, chunk o of it
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_rc + j * STR + OFF + o)),
                 "l"(src + c)
                 : "memory");
  }
  asm volatile("cp.async.commit_group;\n cp.async.wait_group 0;" ::: "memory");
  __syncwarp();
  if constexpr (AGG) {
    if (lane < nw) {
      const double2* u = smem_rc + lane * STR + OFF;
      M G, m;
      cm_load(u, G);
#pragma unroll 4
      for (int i = 1; i < SEG; ++i) {
        cm_load(u + i * W, m);
        G = cm_mul(m, G);
      }
      cm_store(a.agg + (size_t)(g0 + lane) * W, G);
    }
    return;
  }
  const int64_t g = g0 + (lane < nw ? lane : 0), b = g / a.nseg, r = g - b * a.nseg;
  const size_t row = (size_t)(b * (a.k_count + 1) + r * SEG);   // state index of this run's start
  double2* slot = smem_rc + lane * STR;
  if (lane < nw) {
    double pr[D], pi[D];
    const double2* start = a.phi + (size_t)(b * (a.nseg + 1) + r) * D;
#pragma unroll
    for (int d = 0; d < D; ++d) { const double2 v = start[d]; pr[d] = v.x; pi[d] = v.y; }
    double* gJ = a.spin ? a.spin + row * 3 : nullptr;
    if (r == 0) {                                            // ψ_0; a later run's first state is its predecessor's last
      if (a.states)
#pragma unroll
        for (int d = 0; d < D; ++d) __stcs(a.states + row * D + d, make_double2(pr[d], pi[d]));
      if (gJ) {
        double j[3];
        spin_of<D>(pr, pi, j);
        for (int q = 0; q < 3; ++q) __stcs(gJ + q, j[q]);
      }
    }
#pragma unroll 4
    for (int i = 0; i < SEG; ++i) {
      double yr[D], yi[D];
      M m;
      cm_load(slot + OFF + i * W, m);
      cm_apply(m, pr, pi, yr, yi);
#pragma unroll
      for (int d = 0; d < D; ++d) {
        pr[d] = yr[d]; pi[d] = yi[d];
        slot[i * D + d] = make_double2(yr[d], yi[d]);
      }
      if (gJ) {
        double j[3];
        spin_of<D>(pr, pi, j);
        for (int q = 0; q < 3; ++q) __stcs(gJ + (1 + i) * 3 + q, j[q]);
      }
    }
  }
  __syncwarp();
  if (!a.states) return;
  // run j's states ψ[row_j + 1 .. row_j + SEG] are contiguous: one coalesced pass per run
  for (int j = 0; j < nw; ++j) {
    const size_t rj = (size_t)__shfl_sync(0xffffffffu, (long long)row, j);
    double2* dst = a.states + (rj + 1) * D;
    const double2* sj = smem_rc + j * STR;
#pragma unroll
    for (int c = lane; c < SEG * D; c += 32) __stcs(dst + c, sj[c]);
  }
}

template <class M, int SEG, bool AGG = false>
static cudaError_t launch_run_chain(const RunChainArgs& a, cudaStream_t s, int* launches) {
  constexpr size_t smem = run_chain_smem<M, SEG>();
  if constexpr (smem > 48 * 1024) {
    static DeviceCache attr;
    const int dev = current_device();
    if (!attr.get(dev)) {
      const cudaError_t e = cudaFuncSetAttribute(run_chain_kernel<M, SEG, AGG>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      attr.set(dev, 1);
    }
  }
  const int64_t nruns = a.batch * a.nseg;
  run_chain_kernel<M, SEG, AGG><<<(unsigned)((nruns + 31) / 32), 32, smem, s>>>(a);
  ++*launches;
  return cudaGetLastError();
}

// Largest run length the fused path may use with this operator type: a warp's 32 runs fit in shared memory.
template <class M> constexpr int run_max_seg() { return M::W == 2 ? 32 : (M::W == 4 ? 16 : 8); }

template <class M>
static cudaError_t run_segment_chain(int64_t batch, int64_t k_count, int64_t seg, const double* U, const double* phi,
                                     double* states, double* spin, cudaStream_t s, int* launches) {
  if (seg > run_max_seg<M>() || k_count % seg != 0) return cudaErrorInvalidValue;
  const RunChainArgs a{batch, k_count, k_count / seg, reinterpret_cast<const double2*>(U),
                       reinterpret_cast<const double2*>(phi), reinterpret_cast<double2*>(states), spin, nullptr};
  switch (seg) {
    case 4: return launch_run_chain<M, 4>(a, s, launches);
    case 8: return launch_run_chain<M, 8>(a, s, launches);
    case 16: if constexpr (run_max_seg<M>() >= 16) return launch_run_chain<M, 16>(a, s, launches); break;
    case 32: if constexpr (run_max_seg<M>() >= 32) return launch_run_chain<M, 32>(a, s, launches); break;
  }
  return cudaErrorInvalidValue;
}

template <class M>
static cudaError_t run_segment_aggregate(int64_t batch, int64_t k_count, int64_t seg, const double* U, double* agg,
                                         cudaStream_t s, int* launches) {
  if (seg > run_max_seg<M>() || k_count % seg != 0) return cudaErrorInvalidValue;
  const RunChainArgs a{batch, k_count, k_count / seg, reinterpret_cast<const double2*>(U), nullptr, nullptr, nullptr,
                       reinterpret_cast<double2*>(agg)};
  switch (seg) {
    case 4: return launch_run_chain<M, 4, true>(a, s, launches);
    case 8: return launch_run_chain<M, 8, true>(a, s, launches);
    case 16: if constexpr (run_max_seg<M>() >= 16) return launch_run_chain<M, 16, true>(a, s, launches); break;
    case 32: if constexpr (run_max_seg<M>() >= 32) return launch_run_chain<M, 32, true>(a, s, launches); break;
  }
  return cudaErrorInvalidValue;
}

// Run length of the standalone two-pass scan for K intervals (the largest of 32, 16, 8, 4 dividing K with ≥ 2 runs),
// 0 when none applies.
template <class M> static int64_t two_pass_seg(int64_t k_count) {
  for (int64_t c = run_max_seg<M>(); c >= 4; c /= 2)
    if (k_count % c == 0 && k_count >= 2 * c) return c;
  return 0;
}

int fused_max_ipt(int dim, int op_format) {
  if (op_format == OP_SU2) return run_max_seg<SU<2>>();
  return dim == 2 ? run_max_seg<CM<2>>() : run_max_seg<CM<3>>();
}

// Per-sweep product of the tile aggregates, in order: A[b] = T_{n−1} ⋯ T_0.
template <int D>
__global__ void __launch_bounds__(256) combine_tiles_kernel(int64_t tiles_per_sweep, const double2* tiles,
                                                            double2* out) {
  // One block per sweep: thread t multiplies its contiguous run of tile aggregates (later·earlier), a warp shuffle
  // tree and one pass over the 8 warp products give A = T_{n−1} ⋯ T_0.  (Was one thread per sweep walking all
  // n ≈ 4e3 tiles of C4 serially: 0.62 ms; the fixed association is deterministic on every rank.)
  __shared__ CM<D> warp_prod[8];
  const int64_t b = blockIdx.x;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t n = tiles_per_sweep;
  const int64_t per = (n + 255) / 256;
  const int64_t lo = (int64_t)t * per < n ? (int64_t)t * per : n, hi = lo + per < n ? lo + per : n;
  CM<D> A;
  cm_eye(A);
  for (int64_t k = lo; k < hi; ++k) {
    CM<D> T;
    cm_load(tiles + ((size_t)b * n + k) * D * D, T);
    A = cm_mul(T, A);
  }
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const CM<D> B = cm_shfl_down(A, off);
    if ((lane & (2 * off - 1)) == 0) A = cm_mul(B, A);
  }
  if (lane == 0) warp_prod[warp] = A;
  __syncthreads();
  if (t == 0) {
    CM<D> R = warp_prod[0];
    for (int w = 1; w < 8; ++w) R = cm_mul(warp_prod[w], R);
    cm_store(out + (size_t)b * D * D, R);
  }
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

template <int D>
__global__ void spin_projection_kernel(int64_t n, const double2* states, double* out) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  double pr[D], pi[D], j[3];
#pragma unroll
  for (int d = 0; d < D; ++d) { const double2 v = states[s * D + d]; pr[d] = v.x; pi[d] = v.y; }
  spin_of<D>(pr, pi, j);
  out[3 * s + 0] = j[0];
  out[3 * s + 1] = j[1];
  out[3 * s + 2] = j[2];
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

int64_t chain_min_batch() { return kChainMinBatch; }

constexpr int kCoopMaxGrid = 1024;
// Sized for the dense operators of this dim (the compact ones need less).
template <class M> static size_t tile_ws_bytes(int64_t batch, int64_t k_count) {
  return std::max(Scan2Layout<M>(batch, k_count).total, Scan3Layout<M>(batch, k_count, 1).total);
}
// Two-pass (compact operators): [run products: batch·nseg operators][run start states: batch·(nseg + 1)][the coarse
// scan's own workspace for (batch, nseg)].  Sized for the shortest run (4 intervals) whatever K's divisors, so the
// total is monotone in K (the fused path's coarse scan, over K/ipt ≤ K/4 runs, fits the workspace sized for K); only
// below the chain kernel's batch size, the only place the path is taken.
template <class M> static size_t two_pass_ws_bytes(int64_t batch, int64_t k_count) {
  if (batch >= kChainMinBatch || k_count < 8) return 0;
  const int64_t nseg = (k_count + 3) / 4;
  return align256(sizeof(double2) * M::W * (size_t)batch * nseg) +
         align256(sizeof(double2) * M::SD * (size_t)batch * (nseg + 1)) + scan_workspace_bytes(M::SD, batch, nseg);
}
size_t scan_workspace_bytes(int dim, int64_t batch, int64_t k_count) {
  const size_t coop = sizeof(double2) * (size_t)dim * dim * kCoopMaxGrid;
  return std::max({coop,
                   dim == 2 ? std::max(tile_ws_bytes<CM<2>>(batch, k_count), tile_ws_bytes<SU<2>>(batch, k_count))
                            : std::max(tile_ws_bytes<CM<3>>(batch, k_count), tile_ws_bytes<SU<3>>(batch, k_count)),
                   dim == 2 ? two_pass_ws_bytes<SU<2>>(batch, k_count) : two_pass_ws_bytes<SU<3>>(batch, k_count)});
}

// Cooperative small-problem scan (scan_coop_kernel): returns cudaErrorNotSupported when the problem is not eligible.
#ifndef SS_COOP_STAGE_MAX
#define SS_COOP_STAGE_MAX (200 * 1024)   // bytes of operators one CTA stages in shared memory (0: never stage)
#endif
template <class M>
static cudaError_t run_scan_coop(int64_t batch, int64_t k_count, const double* U, const double* psi0, double* states,
                                 double* spin, void* ws, cudaStream_t s, int* launches) {
  constexpr int W = M::W;
  static DeviceCache c_grid, c_stage;   // max co-resident grid + 1 (0: unset); staging available + 1
  const int dev = current_device();
  if (c_grid.get(dev) == 0) {
    int coop = 0, per_sm = 0, max_grid = 0;
    if (cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev) == cudaSuccess && coop &&
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, scan_coop_kernel<M, false>, 128, 0) == cudaSuccess)
      max_grid = std::min(kCoopMaxGrid, device_sms(dev) * std::max(per_sm, 0));
    (void)cudaGetLastError();
    bool stage = SS_COOP_STAGE_MAX > 0 &&
                 cudaFuncSetAttribute(scan_coop_kernel<M, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      SS_COOP_STAGE_MAX) == cudaSuccess;
    if (!stage) (void)cudaGetLastError();                     // staging unavailable: the L2 path only
    c_stage.set(dev, stage ? 2 : 1);
    c_grid.set(dev, max_grid + 1);
  }
  const int max_grid = c_grid.get(dev) - 1;
  const int n_sms = c_stage.get(dev) == 2 ? device_sms(dev) : 0;
  const double bytes = (double)batch * (double)k_count * W * sizeof(double2);
  if (max_grid < 2 || batch * 2 > max_grid || bytes > 64.0 * (1 << 20)) return cudaErrorNotSupported;
  // CTAs per sweep: fill the resident grid, but keep ≥ 256 intervals per CTA
  // (measured: C2's 1e5 intervals prefer 128 CTAs — one predecessor round — C4's 1e6 prefer 256: shorter thread chains)
  const int64_t cap = (k_count > (int64_t)SS_COOP_MAXCPS * 4096) ? 2 * SS_COOP_MAXCPS : SS_COOP_MAXCPS;
  int cps = (int)std::min<int64_t>(std::min<int64_t>(max_grid / batch, cap), (k_count + 255) / 256);
  if (cps < 1) cps = 1;
  CoopArgs a{batch, k_count, cps, reinterpret_cast<const double2*>(U), reinterpret_cast<const double2*>(psi0),
             reinterpret_cast<double2*>(states), spin, static_cast<double2*>(ws)};
  void* args[] = {&a};
  // staged when every CTA has an SM of its own and its run of operators fits the shared-memory budget
  const size_t run_bytes = (size_t)((k_count + cps - 1) / cps) * W * sizeof(double2);
  const bool staged = n_sms > 0 && batch * cps <= n_sms && run_bytes <= (size_t)SS_COOP_STAGE_MAX;
  const cudaError_t e =
      staged ? cudaLaunchCooperativeKernel((const void*)scan_coop_kernel<M, true>, dim3((unsigned)(batch * cps)),
                                           dim3(128), args, run_bytes, s)
             : cudaLaunchCooperativeKernel((const void*)scan_coop_kernel<M, false>, dim3((unsigned)(batch * cps)),
                                           dim3(128), args, 0, s);
  if (e == cudaErrorCooperativeLaunchTooLarge) {   // SMs taken by another context (MPS, green contexts): tile scan
    (void)cudaGetLastError();
    return cudaErrorNotSupported;
  }
  if (e == cudaSuccess) ++*launches;
  return e;
}

size_t aggregate_workspace_bytes(int dim, int64_t batch, int64_t k_count) {
  // v1 tiling; per-tile totals live in the workspace, then one combine per sweep
  return dim == 2 ? scan_ws_bytes<2>(batch, k_count) : scan_ws_bytes<3>(batch, k_count);
}

template <int D>
static cudaError_t run_aggregate(int64_t batch, int64_t k_count, const double* U, double* aggregate, void* ws,
                                 cudaStream_t s, int* launches) {
  ScanLayout<D> L(batch, k_count);
  ScanArgs a;
  a.batch = batch;
  a.k_count = k_count;
  a.tiles_per_sweep = L.tiles_per_sweep;
  a.U = reinterpret_cast<const double2*>(U);
  a.aggregate_out = reinterpret_cast<double2*>(static_cast<char*>(ws) + L.off_agg);
  if (L.ntiles > 0x7fffffffLL) return cudaErrorInvalidValue;
  constexpr size_t smem = sizeof(double2) * (size_t)tile_size<D>() * D * D;
  static DeviceCache attr;
  const int dev = current_device();
  if (!attr.get(dev)) {
    const cudaError_t e = cudaFuncSetAttribute(aggregate_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr.set(dev, 1);
  }
  aggregate_kernel<D><<<(unsigned)L.ntiles, kScanThreads, smem, s>>>(a);
  ++*launches;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  combine_tiles_kernel<D><<<(unsigned)batch, 256, 0, s>>>(L.tiles_per_sweep, a.aggregate_out,
                                                          reinterpret_cast<double2*>(aggregate));
  ++*launches;
  return cudaGetLastError();
}

template <class M>
static cudaError_t run_scan2(int64_t batch, int64_t k_count, const double* U, const double* psi0, double* states,
                             double* spin, void* ws, cudaStream_t s, int* launches) {
  Scan2Layout<M> L(batch, k_count);
  char* w = static_cast<char*>(ws);
  Scan2Args a;
  a.batch = batch;
  a.k_count = k_count;
  a.tiles_per_sweep = L.tiles_per_sweep;
  a.ntiles = L.ntiles;
  a.U = reinterpret_cast<const double2*>(U);
  a.psi0 = reinterpret_cast<const double2*>(psi0);
  a.states = reinterpret_cast<double2*>(states);
  a.spin = spin;
  a.ticket = reinterpret_cast<unsigned long long*>(w);
  a.flags = reinterpret_cast<int*>(w + L.off_flags);
  a.agg = reinterpret_cast<double2*>(w + L.off_agg);
  a.psi_end = reinterpret_cast<double2*>(w + L.off_psi);
  cudaError_t e = cudaMemsetAsync(w, 0, L.off_agg, s);   // ticket + flags
  if (e != cudaSuccess) return e;
  constexpr size_t smem = scan2_smem<M>();
  static DeviceCache c_grid;
  const int dev = current_device();
  int grid = c_grid.get(dev);
  if (grid == 0) {
    e = cudaFuncSetAttribute(scan2_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, scan2_kernel<M>, Scan2Cfg<M>::NT, smem);
    if (e != cudaSuccess) return e;
    grid = device_sms(dev) * (per_sm > 0 ? per_sm : 1);   // persistent: every CTA resident (look-back forward progress)
    c_grid.set(dev, grid);
  }
  const int g = (int)std::min<int64_t>(grid, L.ntiles);
  scan2_kernel<M><<<g, Scan2Cfg<M>::NT, smem, s>>>(a);
  ++*launches;
  return cudaGetLastError();
}

template <class M> static int scan3_nst(int64_t batch, int64_t k_count, int grid) {
  int nst = Scan3Cfg<M>::MAXST;   // largest tile that still leaves ≥ 4 tiles per CTA
  while (nst > 1 && Scan3Layout<M>(batch, k_count, nst).ntiles < 4LL * grid) nst >>= 1;
  return nst;
}

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// 4-D view of a [B][rows·IPT + …][w] complex128 array (w = W double2 per operator, D per state) for scan3's stage
// boxes: dim0 = the C·w·2 doubles of one stage of one row, dim1 = stage s, dim2 = row (IPT intervals), dim3 = sweep.
// The box is one double2 wider than dim0: the out-of-bounds element is zero-filled on loads and dropped on stores,
// and gives the shared-memory rows an odd 16-B pitch.
static cudaError_t encode_stage_map(CUtensorMap* tm, const void* base, int w, int C, int nst, int64_t rows,
                                    int64_t sweep_stride_items, int64_t batch, int box_rows) {
  static std::atomic<EncodeTiled> encode{nullptr};
  EncodeTiled fn = encode.load();
  if (!fn) {
    cudaDriverEntryPointQueryResult qr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&fn, cudaEnableDefault, &qr);
    if (e != cudaSuccess || qr != cudaDriverEntryPointSuccess || !fn) return cudaErrorSymbolNotFound;
    encode.store(fn);
  }
  const cuuint64_t item = (cuuint64_t)w * sizeof(double2);
  const cuuint64_t dims[4] = {(cuuint64_t)C * w * 2, (cuuint64_t)nst, (cuuint64_t)rows, (cuuint64_t)batch};
  const cuuint64_t strides[3] = {C * item, (cuuint64_t)nst * C * item, (cuuint64_t)sweep_stride_items * item};
  const cuuint32_t box[4] = {(cuuint32_t)(C * w * 2 + 2), 1u, (cuuint32_t)box_rows, 1u};
  const cuuint32_t estr[4] = {1u, 1u, 1u, 1u};
  const CUresult r = fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// persistent grid of scan3 on the current device: every CTA resident (look-back forward progress); 0 on error
template <class M> static int scan3_grid() {
  static DeviceCache c_grid;
  const int dev = current_device();
  int grid = c_grid.get(dev);
  if (grid == 0) {
    if (cudaFuncSetAttribute(scan3_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)scan3_smem<M>()) !=
        cudaSuccess)
      return 0;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, scan3_kernel<M>, Scan3Cfg<M>::NT, scan3_smem<M>()) !=
        cudaSuccess)
      return 0;
    grid = device_sms(dev) * (per_sm > 0 ? per_sm : 1);
    c_grid.set(dev, grid);
  }
  return grid;
}

template <class M>
static cudaError_t run_scan3(int64_t batch, int64_t k_count, const double* U, const double* psi0, double* states,
                             double* spin, void* ws, cudaStream_t s, int* launches) {
  using Cfg = Scan3Cfg<M>;
  constexpr int D = M::SD;
  constexpr size_t smem = scan3_smem<M>();
  const int grid = scan3_grid<M>();
  if (grid == 0) return cudaErrorInvalidConfiguration;
  cudaError_t e;
  const int nst = scan3_nst<M>(batch, k_count, grid);
  Scan3Layout<M> L(batch, k_count, nst);
  char* w = static_cast<char*>(ws);
  Scan3Args A3;
  Scan2Args& a = A3.s;
  A3.nst = nst;
  a.batch = batch;
  a.k_count = k_count;
  a.tiles_per_sweep = L.tiles_per_sweep;
  a.ntiles = L.ntiles;
  a.U = reinterpret_cast<const double2*>(U);
  a.psi0 = reinterpret_cast<const double2*>(psi0);
  a.states = reinterpret_cast<double2*>(states);
  a.spin = spin;
  a.ticket = reinterpret_cast<unsigned long long*>(w);
  a.flags = reinterpret_cast<int*>(w + L.off_flags);
  a.agg = reinterpret_cast<double2*>(w + L.off_agg);
  a.psi_end = reinterpret_cast<double2*>(w + L.off_psi);
  CUtensorMap tmU, tmS;
  std::memset(&tmU, 0, sizeof tmU);
  std::memset(&tmS, 0, sizeof tmS);
  const int64_t ipt = (int64_t)nst * Cfg::C, rows = k_count / ipt;
  A3.tensor_u = k_count >= L.tile;             // some tile is full
  A3.tensor_s = A3.tensor_u && states != nullptr;
  if (A3.tensor_u) {
    e = encode_stage_map(&tmU, U, M::W, Cfg::C, nst, rows, k_count, batch, Cfg::NT);
    if (e != cudaSuccess) return e;
  }
  if (A3.tensor_s) {   // states[b][k + 1] for interval k: base at state 1, sweep stride K + 1
    e = encode_stage_map(&tmS, states + 2 * D, D, Cfg::C, nst, rows, k_count + 1, batch, 32);   // per-warp boxes
    if (e != cudaSuccess) return e;
  }
  e = cudaMemsetAsync(w, 0, L.off_agg, s);   // ticket + flags
  if (e != cudaSuccess) return e;
  const int g = (int)std::min<int64_t>(grid, L.ntiles);
  scan3_kernel<M><<<g, Cfg::NT, smem, s>>>(A3, tmU, tmS);
  ++*launches;
  return cudaGetLastError();
}

template <class M>
static cudaError_t run_state_scan(int64_t batch, int64_t k_count, const double* U, const double* psi0, double* states,
                                  void* ws, cudaStream_t s, int* launches, double* spin);

// Standalone two-pass scan for compact SU(2) operators (reduce-then-scan, the fused path's structure with its first
// pass as a kernel of its own): run products of `seg` consecutive operators (run_chain_kernel, AGG), a coarse scan of
// them into the run start states, then the run chain — U read twice, each time by a plain coalesced stream, instead
// of through a look-back tile scan.  cudaErrorNotSupported when no run length divides K.
template <class M>
static cudaError_t run_two_pass(int64_t batch, int64_t k_count, const double* U, const double* psi0, double* states,
                                double* spin, void* ws, cudaStream_t s, int* launches) {
  const int64_t seg = two_pass_seg<M>(k_count);
  if (!seg) return cudaErrorNotSupported;
  const int64_t nseg = k_count / seg;
  char* w = static_cast<char*>(ws);
  double* agg = reinterpret_cast<double*>(w);
  w += align256(sizeof(double2) * M::W * (size_t)batch * nseg);
  double* phi = reinterpret_cast<double*>(w);
  w += align256(sizeof(double2) * M::SD * (size_t)batch * (nseg + 1));
  cudaError_t e = run_segment_aggregate<M>(batch, k_count, seg, U, agg, s, launches);
  if (e != cudaSuccess) return e;
  e = run_state_scan<M>(batch, nseg, agg, psi0, phi, w, s, launches, nullptr);
  if (e != cudaSuccess) return e;
  return run_segment_chain<M>(batch, k_count, seg, U, phi, states, spin, s, launches);
}

// Path override for tests and measurement tools: SPINSIM_SCAN_PATH = coop | chain | scan2 | scan3 | twopass forces
// that kernel (coop and chain only where they apply: coop needs an L2-sized problem; twopass compact operators and a
// run length dividing K); unset = the heuristic below.  Read on every call (one getenv per scan launch), so a test
// can switch paths within one process.
static int forced_scan_path() {
  const char* p = std::getenv("SPINSIM_SCAN_PATH");
  if (!p) return 0;
  const char* names[] = {"", "coop", "chain", "scan2", "scan3", "twopass"};
  for (int i = 1; i < 6; ++i)
    if (!std::strcmp(p, names[i])) return i;
  return 0;
}

// Path choice: the cooperative single-wave scan for L2-sized problems; the per-sweep chain for ≥ chain_min_batch_of
// sweeps; otherwise compact SU(2) operators take the two-pass scan where a run length divides K, dense ones scan3
// where its tiles get ≥ 4 stages (long sweeps, moderate batch) and scan2 for the rest.
template <class M>
static cudaError_t run_state_scan(int64_t batch, int64_t k_count, const double* U, const double* psi0, double* states,
                                  void* ws, cudaStream_t s, int* launches, double* spin) {
  switch (forced_scan_path()) {
    case 1: {
      const cudaError_t e = run_scan_coop<M>(batch, k_count, U, psi0, states, spin, ws, s, launches);
      if (e != cudaErrorNotSupported) return e;
      break;
    }
    case 2: return run_chain<M>(batch, k_count, U, psi0, states, spin, s, launches);
    case 3: return run_scan2<M>(batch, k_count, U, psi0, states, spin, ws, s, launches);
    case 4: return run_scan3<M>(batch, k_count, U, psi0, states, spin, ws, s, launches);
    case 5:
      if constexpr (M::W == 2) {
        const cudaError_t e = run_two_pass<M>(batch, k_count, U, psi0, states, spin, ws, s, launches);
        if (e != cudaErrorNotSupported) return e;
      }
      break;
  }
  const cudaError_t e = run_scan_coop<M>(batch, k_count, U, psi0, states, spin, ws, s, launches);
  if (e != cudaErrorNotSupported) return e;
  if (batch >= chain_min_batch_of<M>()) return run_chain<M>(batch, k_count, U, psi0, states, spin, s, launches);
  if constexpr (M::W == 2) {
    const cudaError_t e2 = run_two_pass<M>(batch, k_count, U, psi0, states, spin, ws, s, launches);
    if (e2 != cudaErrorNotSupported) return e2;
  }
  // scan3 amortises its look-back over big tiles; below ~4 stages per tile (small problems) scan2's single pass wins
  if (scan3_nst<M>(batch, k_count, scan3_grid<M>()) >= 4)
    return run_scan3<M>(batch, k_count, U, psi0, states, spin, ws, s, launches);
  return run_scan2<M>(batch, k_count, U, psi0, states, spin, ws, s, launches);
}

cudaError_t launch_scan(int dim, int64_t batch, int64_t k_count, const double* U, const double* psi0, double* states,
                        void* ws, cudaStream_t s, int* launches, double* spin, int op_format) {
  if (op_format == OP_SU2)
    return dim == 2 ? run_state_scan<SU<2>>(batch, k_count, U, psi0, states, ws, s, launches, spin)
                    : run_state_scan<SU<3>>(batch, k_count, U, psi0, states, ws, s, launches, spin);
  return dim == 2 ? run_state_scan<CM<2>>(batch, k_count, U, psi0, states, ws, s, launches, spin)
                  : run_state_scan<CM<3>>(batch, k_count, U, psi0, states, ws, s, launches, spin);
}

// Fused path (the interval kernel wrote run aggregates G[b][r] = U_{(r+1)seg−1} ⋯ U_{r·seg}): the coarse scan turns
// them into the run start states phi[b][r] = G[b][r−1] ⋯ G[b][0] ψ0[b] (any state-scan path, on 1/seg of the data),
// then one chain thread per run applies the run's own operators from phi[b][r] — every run independent, so the
// states pass is a plain stream over U (read once) and ψ (written once).
template <class M>
static cudaError_t run_fused(int64_t batch, int64_t k_count, int64_t seg, const double* U, const double* run_agg,
                             const double* psi0, double* phi, double* states, void* ws, cudaStream_t s, int* launches,
                             double* spin) {
  const int64_t nseg = (k_count + seg - 1) / seg;
  cudaError_t e = run_state_scan<M>(batch, nseg, run_agg, psi0, phi, ws, s, launches, nullptr);
  if (e != cudaSuccess) return e;
  return run_segment_chain<M>(batch, k_count, seg, U, phi, states, spin, s, launches);
}

cudaError_t launch_fused_scan(int dim, int64_t batch, int64_t k_count, int64_t seg, const double* U,
                              const double* run_agg, const double* psi0, double* phi, double* states, void* ws,
                              cudaStream_t s, int* launches, double* spin, int op_format) {
  if (op_format == OP_SU2)
    return dim == 2 ? run_fused<SU<2>>(batch, k_count, seg, U, run_agg, psi0, phi, states, ws, s, launches, spin)
                    : run_fused<SU<3>>(batch, k_count, seg, U, run_agg, psi0, phi, states, ws, s, launches, spin);
  return dim == 2 ? run_fused<CM<2>>(batch, k_count, seg, U, run_agg, psi0, phi, states, ws, s, launches, spin)
                  : run_fused<CM<3>>(batch, k_count, seg, U, run_agg, psi0, phi, states, ws, s, launches, spin);
}

cudaError_t launch_aggregate(int dim, int64_t batch, int64_t k_count, const double* U, double* aggregate, void* ws,
                             cudaStream_t s, int* launches) {
  return dim == 2 ? run_aggregate<2>(batch, k_count, U, aggregate, ws, s, launches)
                  : run_aggregate<3>(batch, k_count, U, aggregate, ws, s, launches);
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
