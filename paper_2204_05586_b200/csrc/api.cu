// api.cu — the C ABI declared in include/spinsim_b200.h: validation, planning, workspace layout and launches.
// Host code only; the arithmetic of the method lives in the kernels (interval_*.cu, scan.cu).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/spinsim_b200.h"
#include "dispatch.h"
#include "interval_kernel.cuh"
#include "kernels.h"
#include "user_field.h"

namespace {

thread_local std::string g_err;
std::atomic<int64_t> g_launches{0};

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(SS_ERR_CUDA, "%s: CUDA error %d (%s)", where, (int)e, cudaGetErrorString(e));
}

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// cudaMemcpy2DAsync rejects pitches above the device's cudaDevAttrMaxPitch (≈ 2^31 B: spin-one states of one sweep
// past ≈ 45M intervals); beyond it the rows go as one cudaMemcpyAsync each.
cudaError_t copy_rows(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height,
                      cudaMemcpyKind kind, cudaStream_t st) {
  static std::atomic<long long> max_pitch{0};
  long long mp = max_pitch.load(std::memory_order_relaxed);
  if (mp == 0) {
    int dev = 0, v = 0;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetAttribute(&v, cudaDevAttrMaxPitch, dev) == cudaSuccess && v > 0)
      mp = v;
    else
      mp = 1LL << 31;
    max_pitch.store(mp, std::memory_order_relaxed);
  }
  if (height == 1 || ((long long)dpitch <= mp && (long long)spitch <= mp))
    return height == 1 ? cudaMemcpyAsync(dst, src, width, kind, st)
                       : cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, kind, st);
  for (size_t r = 0; r < height; ++r) {
    const cudaError_t e = cudaMemcpyAsync(static_cast<char*>(dst) + r * dpitch,
                                          static_cast<const char*>(src) + r * spitch, width, kind, st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

int field_params(int field) {
  switch (field) {
    case SS_FIELD_CONSTANT: return 4;
    case SS_FIELD_RABI_LINEAR: return 2;
    case SS_FIELD_RABI_CIRCULAR: return 2;
    case SS_FIELD_NEURAL: return 7;
    case SS_FIELD_GRADIENT: return 2;
    case SS_FIELD_SU3_CONSTANT: return 8;
    case SS_FIELD_SU3_DRIVE: return 6;
  }
  return -1;
}

bool is_su3_field(int field) { return field == SS_FIELD_SU3_CONSTANT || field == SS_FIELD_SU3_DRIVE; }

// Column of the sweep table holding ω_q (must be 0 for the analytic spin-one exponentiator), or −1.
int qcol_of(int field) {
  switch (field) {
    case SS_FIELD_CONSTANT: return 3;
    case SS_FIELD_NEURAL: return 6;
  }
  return -1;
}

}  // namespace

struct ss_sim {
  ss_sim_desc d;
  int dim = 0;
  int P = 0;
  int validate = 1;
  ssb::IntervalLaunchFn interval = nullptr;
  ssb::ExpoLaunchFn expo = nullptr;
  bool user = false;               // run-time compiled user field (ss_create_user)
  ssb::UserKernel user_kernel;
  // ss_evaluate_host pipeline: streams[0] computes, streams[1] copies, streams[2] scans the time chunks (so chunk c's
  // scan overlaps chunk c+1's interval kernel); three staging slots; events order them
  cudaStream_t streams[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t split_event = nullptr;  // ss_set_split_event: recorded by ss_evaluate between interval kernel and scan
  static constexpr int kSlots = 3;
  cudaEvent_t computed[kSlots] = {};   // slot's kernels done → its D2H may start
  cudaEvent_t drained[kSlots] = {};    // slot's D2H done → its buffers may be reused
  cudaEvent_t stepped[kSlots] = {};    // slot's interval kernel done → its scan may start
  int device = -1;
  struct Slot {
    void* buf = nullptr;
    size_t cap = 0;
  } slots[kSlots], aux;   // aux: sweep table + running carry of the time-chunked pipeline
};

namespace {

ssb::IntervalLaunchFn pick_interval(const ss_sim_desc& d) {
  const bool f32 = d.precision == SS_FP32;
  if (d.spin == SS_SPIN_HALF)
    return f32 ? ssb::interval_table_half_f32(d.integration, d.field) : ssb::interval_table_half_f64(d.integration, d.field);
  if (d.exponentiation == SS_EXP_LIE_TROTTER)
    return f32 ? ssb::interval_table_one_lt_f32(d.integration, d.field)
               : ssb::interval_table_one_lt_f64(d.integration, d.field);
  if (d.exponentiation == SS_EXP_LIE_TROTTER_SU3)
    return f32 ? ssb::interval_table_one_su3_f32(d.integration, d.field)
               : ssb::interval_table_one_su3_f64(d.integration, d.field);
  return f32 ? ssb::interval_table_one_an_f32(d.integration, d.field) : ssb::interval_table_one_an_f64(d.integration, d.field);
}

ssb::MagnusLaunchFn pick_magnus(const ss_sim_desc& d) {
  const bool f32 = d.precision == SS_FP32;
  if (d.spin == SS_SPIN_HALF) return f32 ? ssb::magnus_table_half_f32(d.field) : ssb::magnus_table_half_f64(d.field);
  if (d.exponentiation == SS_EXP_LIE_TROTTER)
    return f32 ? ssb::magnus_table_one_lt_f32(d.field) : ssb::magnus_table_one_lt_f64(d.field);
  if (d.exponentiation == SS_EXP_LIE_TROTTER_SU3)
    return f32 ? ssb::magnus_table_one_su3_f32(d.field) : ssb::magnus_table_one_su3_f64(d.field);
  return f32 ? ssb::magnus_table_one_an_f32(d.field) : ssb::magnus_table_one_an_f64(d.field);
}

ssb::ExpoLaunchFn pick_expo(const ss_sim_desc& d) {
  const bool f32 = d.precision == SS_FP32;
  if (d.spin == SS_SPIN_HALF) return f32 ? ssb::expo_table_half_f32() : ssb::expo_table_half_f64();
  if (d.exponentiation == SS_EXP_LIE_TROTTER) return f32 ? ssb::expo_table_one_lt_f32() : ssb::expo_table_one_lt_f64();
  if (d.exponentiation == SS_EXP_LIE_TROTTER_SU3)
    return f32 ? ssb::expo_table_one_su3_f32() : ssb::expo_table_one_su3_f64();
  return f32 ? ssb::expo_table_one_an_f32() : ssb::expo_table_one_an_f64();
}

int plan_grid(double t0, double t1, double dt_int, double dt_out, int64_t* K, int64_t* L, double* dt) {
  if (!std::isfinite(t0) || !std::isfinite(t1) || !std::isfinite(dt_int) || !std::isfinite(dt_out))
    return fail(SS_ERR_NONFINITE, "time arguments must be finite");
  if (!(t1 > t0)) return fail(SS_ERR_INVALID, "time_end (%g) must exceed time_start (%g)", t1, t0);
  if (!(dt_int > 0)) return fail(SS_ERR_INVALID, "time_step_integration must be > 0");
  if (!(dt_out > 0)) return fail(SS_ERR_INVALID, "time_step_output must be > 0");
  const double kf = (t1 - t0) / dt_out, lf = dt_out / dt_int;
  if (kf > 9.0e15 || lf > 9.0e15) return fail(SS_ERR_INVALID, "time grid too large");
  const long long k = std::llround(kf), l = std::llround(lf);
  if (k < 1 || std::fabs(kf - (double)k) > 1e-9 * kf)
    return fail(SS_ERR_INVALID, "(time_end - time_start)/time_step_output = %.17g is not an integer", kf);
  if (l < 1 || std::fabs(lf - (double)l) > 1e-9 * lf)
    return fail(SS_ERR_INVALID, "time_step_output/time_step_integration = %.17g is not an integer", lf);
  *K = k;
  *L = l;
  *dt = dt_out / (double)l;
  return SS_OK;
}

// Sub-interval split (DESIGN.md §5 item 8): S = 1, 2, 4, … ≤ 32 adjacent lanes share an interval (S | L), each
// running L/S fine steps.  S minimises the modelled time ⌈n·S/R⌉ · (L/S + c0 + c1·log2 S): n intervals, R resident
// threads (SMs × resident blocks × 128), c0 the per-thread setup and c1 the per-level combine cost in fine steps
// (short SU(2)-form steps: 2.5 / 0.17; 3×3 Lie–Trotter steps: 0.15 / 0.03).  n is the WHOLE problem (batch × K of
// the grid), never the launched part, so partitions and host-API chunks pick the same S and reproduce the same
// operators bit for bit.  C4 (1e6 intervals × 1000 steps): S = 4, 14 → 53 rounds of a quarter the length (−4.5 %).
#ifndef SS_FORCE_SPLIT
#define SS_FORCE_SPLIT 0    // tuning experiments only: a fixed S (must divide L)
#endif
// Interval-kernel threads resident on the device at once (one wave).
// SM counts are cached per device ordinal (a process may drive several GPUs); 148 when no device answers
// (host-only planning, e.g. ss_host_chunk_plan on a machine without a GPU).
double resident_threads(const ss_sim* s) {
  static std::atomic<int> sms_of[64];
  int dev = -1, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = -1;
  if (dev >= 0) sms = sms_of[dev].load(std::memory_order_relaxed);
  if (sms == 0) {
    if (dev >= 0 && cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && sms > 0) {
      sms_of[dev].store(sms, std::memory_order_relaxed);
    } else {
      sms = 148;
      (void)cudaGetLastError();
    }
  }
  const bool su3 = s->d.exponentiation == SS_EXP_LIE_TROTTER_SU3;
  return (double)sms * (su3 ? SS_INTERVAL_MINBLOCKS_SU3 : SS_INTERVAL_MINBLOCKS) * ssb::kIntervalThreads;
}

int choose_split(const ss_sim* s, int64_t n_total, int64_t L) {
  if (SS_FORCE_SPLIT > 0 && L % SS_FORCE_SPLIT == 0) return SS_FORCE_SPLIT;
  const bool short_steps = s->dim == 2 || s->d.exponentiation == SS_EXP_ANALYTIC;
  const double R = resident_threads(s);
  const double c0 = short_steps ? 2.5 : 0.15, c1 = short_steps ? 0.17 : 0.03;
  int best = 1;
  double best_t = 0.0;
  for (int S = 1, lev = 0; S <= 32 && L % S == 0; S *= 2, ++lev) {
    const double t = std::ceil((double)n_total * S / R) * ((double)L / S + c0 + c1 * lev);
    if (S == 1 || t < best_t * 0.995) { best = S; best_t = t; }
  }
  return best;
}

ssb::IntervalParams make_params(const ss_sim* s, double t0, double dt_out, double dt, int64_t L, int64_t k_begin,
                                int64_t k_count, int64_t batch, const double* sweep, double* U, int64_t n_total) {
  ssb::IntervalParams p;
  p.t0 = t0;
  p.dt_out = dt_out;
  p.dt = dt;
  p.g1dt = ssb::kG1 * dt;      // host IEEE double multiply: fl(g1·δt) (reading R7)
  p.g2dt = ssb::kG2 * dt;
  p.half_dt = 0.5 * dt;
  p.half_dt_out = 0.5 * dt_out;
  p.wpd = ssb::kWPlus * dt;
  p.wmd = ssb::kWMinus * dt;
  p.L = L;
  p.k_begin = k_begin;
  p.k_count = k_count;
  p.batch = batch;
  p.n_threads = batch * k_count;
  p.k_stride = k_count;
  p.ipt = 1;
  p.run_agg = nullptr;
  p.tau = s->d.trotter_cutoff;
  p.frame = s->d.use_rotating_frame;
  p.split = choose_split(s, n_total, L);
  p.op_format = ssb::OP_DENSE;
  p.sweep = sweep;
  p.unitaries = U;
  return p;
}

// The SU(2)-form paths (spin-half; analytic spin-one accumulated in SU(2), DESIGN.md §5 items 10-11) can hand their
// operators to the scan as SU(2) elements (32 B per interval instead of 64 / 144 B) when U_k is not an output.
bool su2_form(const ss_sim* s) { return s->dim == 2 || s->d.exponentiation == SS_EXP_ANALYTIC; }

int check_device_ptr(const void* p, const char* name) {
  if (!p) return fail(SS_ERR_INVALID, "%s is NULL", name);
  if ((reinterpret_cast<uintptr_t>(p) & 15) != 0) return fail(SS_ERR_INVALID, "%s must be 16-byte aligned", name);
  return SS_OK;
}

int ensure_device() {
  int n = 0;
  const cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) return fail(SS_ERR_CUDA, "no CUDA device available (no CPU fallback exists)");
  return SS_OK;
}

int launch_interval_checked(ss_sim* s, const ssb::IntervalParams& p, cudaStream_t st) {
  const cudaError_t e = s->user ? ssb::launch_user(s->user_kernel, p, st) : s->interval(p, st);
  if (e != cudaSuccess) return cuda_fail(e, "interval kernel launch");
  g_launches.fetch_add(1);
  return SS_OK;
}

// Fused run aggregates (DESIGN.md §5 item 16): for long problems (S = 1, ≥ 16 waves of interval threads even at 4
// intervals per thread) each interval-kernel thread computes ipt consecutive intervals and multiplies their U_k into
// a run aggregate; a coarse scan over the aggregates gives every run's start state and one chain lane per run
// writes the states — U_k is read once, by a plain streaming pass, instead of through a look-back tile scan.  ipt is
// the largest of 32, 16, 8, 4 that divides K, fits the operator type (ssb::fused_max_ipt: a warp's 32 runs in shared
// memory) and keeps ≥ 16 waves.  Below the chain kernel's batch size only (it streams U once
// already); the workspace holds ≤ ⌈K/4⌉ run aggregates + ⌈K/4⌉ + 1 run states per sweep.
// SPINSIM_FUSED=0 turns it off, SPINSIM_FUSED_IPT=n forces ipt (comparison runs; read on every call).
constexpr int64_t kFusedMinIpt = 4;
constexpr double kFusedMinWaves = 16.0;
bool fused_batch(int64_t batch) { return batch < ssb::chain_min_batch(); }
size_t fused_bytes(int dim, int64_t batch, int64_t K) {
  if (!fused_batch(batch)) return 0;
  const size_t nseg = (size_t)((K + kFusedMinIpt - 1) / kFusedMinIpt);
  return align256(sizeof(double) * 2 * dim * dim * (size_t)batch * nseg) +
         align256(sizeof(double) * 2 * dim * (size_t)batch * (nseg + 1));
}
// ipt of the fused path for this launch, 0 = unfused
int64_t fused_ipt(const ss_sim* s, int64_t batch, int64_t K, int S, int op_format) {
  const char* env = std::getenv("SPINSIM_FUSED");
  if ((env && env[0] == '0') || !fused_batch(batch) || S != 1) return 0;
  const int64_t max_ipt = ssb::fused_max_ipt(s->dim, op_format);
  const char* fi = std::getenv("SPINSIM_FUSED_IPT");
  if (fi) {
    const int64_t v = std::atoll(fi);
    return (v >= kFusedMinIpt && v <= max_ipt && (v & (v - 1)) == 0 && K % v == 0 && K >= 2 * v) ? v : 0;
  }
  // Dense 3×3 operators (Lie–Trotter, su(3), analytic spin-one with U requested): the run products cost the interval
  // kernel more than the streamed states pass saves (measured: C3's 1024-sweep shard −0.8 %, C5 Lie–Trotter −0.2 %,
  // G1 shard −3 %, profiles/r02/s32_dense/), so only SPINSIM_FUSED_IPT takes them fused.
  if (s->dim == 3 && op_format != ssb::OP_SU2) return 0;
  const double R = resident_threads(s);
  for (int64_t ipt = max_ipt; ipt >= kFusedMinIpt; ipt /= 2)
    if (K % ipt == 0 && (double)batch * (double)(K / ipt) >= kFusedMinWaves * R) return ipt;
  return 0;
}
// Sets up the interval launch for the fused path: one thread slot per ipt intervals, run aggregates at `agg`.
void enable_fused(ssb::IntervalParams& p, int64_t ipt, double* agg) {
  p.ipt = ipt;
  p.k_stride = (p.k_count + ipt - 1) / ipt;
  p.n_threads = p.batch * p.k_stride;
  p.run_agg = agg;
}
// Where the fused path's run aggregates and run states live inside the ss_evaluate workspace region `fw`.
double* fused_phi(char* fw, int dim, int64_t batch, int64_t K) {
  return reinterpret_cast<double*>(
      fw + align256(sizeof(double) * 2 * dim * dim * (size_t)batch * (size_t)((K + kFusedMinIpt - 1) / kFusedMinIpt)));
}

// Interval kernel for p, then the state propagation from d_psi0 into d_states (row a9): fused (run aggregates +
// coarse scan + run chain) where fused_ipt allows it and the caller has a fused region `fused_ws`, else the state-scan
// heuristic in scan_ws.  The scan runs on `scan_st`; when that is not `cs`, `stepped` orders it after the interval
// kernel.  `split_event` (profiling) is recorded between the two.
int launch_path(ss_sim* s, ssb::IntervalParams& p, const double* d_psi0, double* d_states, void* scan_ws,
                char* fused_ws, cudaStream_t cs, cudaStream_t scan_st, cudaEvent_t stepped) {
  const int64_t ipt = fused_ws ? fused_ipt(s, p.batch, p.k_count, p.split, p.op_format) : 0;
  if (ipt) enable_fused(p, ipt, reinterpret_cast<double*>(fused_ws));
  int rc = launch_interval_checked(s, p, cs);
  if (rc) return rc;
  cudaError_t e;
  if (s->split_event && (e = cudaEventRecord(s->split_event, cs)) != cudaSuccess) return cuda_fail(e, "split event record");
  if (scan_st != cs && ((e = cudaEventRecord(stepped, cs)) || (e = cudaStreamWaitEvent(scan_st, stepped, 0))))
    return cuda_fail(e, "event record/wait");
  int n = 0;
  e = ipt ? ssb::launch_fused_scan(s->dim, p.batch, p.k_count, ipt, p.unitaries, p.run_agg, d_psi0,
                                   fused_phi(fused_ws, s->dim, p.batch, p.k_count), d_states, scan_ws, scan_st, &n,
                                   nullptr, p.op_format)
          : ssb::launch_scan(s->dim, p.batch, p.k_count, p.unitaries, d_psi0, d_states, scan_ws, scan_st, &n, nullptr,
                             p.op_format);
  g_launches.fetch_add(n);
  return e == cudaSuccess ? SS_OK : cuda_fail(e, "scan launch");
}

}  // namespace

extern "C" {

int ss_version(void) { return 102; }

int ss_num_coefficients(const ss_sim* s) {
  if (!s) return fail(SS_ERR_INVALID, "sim is NULL");
  return s->d.exponentiation == SS_EXP_LIE_TROTTER_SU3 ? 8 : 4;
}

const char* ss_last_error(void) { return g_err.c_str(); }

int64_t ss_kernel_launches(void) { return g_launches.load(); }

int ss_num_sweep_params(int32_t field) { return field_params(field); }

int ss_create(const ss_sim_desc* desc, ss_sim** out) {
  if (!desc || !out) return fail(SS_ERR_INVALID, "desc and out must be non-NULL");
  const ss_sim_desc& d = *desc;
  if (d.spin != SS_SPIN_HALF && d.spin != SS_SPIN_ONE) return fail(SS_ERR_INVALID, "spin must be 1 (half) or 2 (one), got %d", d.spin);
  if (d.integration < SS_CF4 || d.integration > SS_HEUN) return fail(SS_ERR_INVALID, "integration %d unknown", d.integration);
  if (d.exponentiation != SS_EXP_ANALYTIC && d.exponentiation != SS_EXP_LIE_TROTTER &&
      d.exponentiation != SS_EXP_LIE_TROTTER_SU3)
    return fail(SS_ERR_INVALID, "exponentiation %d unknown", d.exponentiation);
  if (d.spin == SS_SPIN_HALF && d.exponentiation != SS_EXP_ANALYTIC)
    return fail(SS_ERR_UNSUPPORTED, "spin-half uses the analytic SU(2) exponentiator (P:359); Lie-Trotter is spin-one only");
  if (is_su3_field(d.field) && d.exponentiation != SS_EXP_LIE_TROTTER_SU3)
    return fail(SS_ERR_UNSUPPORTED, "field %d has U1/U2/V1/V2 components: it needs SS_EXP_LIE_TROTTER_SU3", d.field);
  if (d.trotter_cutoff < 0 || d.trotter_cutoff > 60) return fail(SS_ERR_INVALID, "trotter_cutoff %d outside 0..60", d.trotter_cutoff);
  if (d.use_rotating_frame != 0 && d.use_rotating_frame != 1) return fail(SS_ERR_INVALID, "use_rotating_frame must be 0 or 1");
  if (d.precision != SS_FP64 && d.precision != SS_FP32) return fail(SS_ERR_INVALID, "precision %d unknown", d.precision);
  // FP32 mode's 1e-4 bar (BASELINE north_star) holds in the rotating frame it is built for: in the lab
  // frame every fine step rotates by |ω_z δt| ~ 1 rad and the FP32 rounding accumulates as ε₃₂·Σ|a| (4.5e-4 after
  // 300 intervals) — so the combination is refused rather than run below its bar.
  if (d.precision == SS_FP32 && !d.use_rotating_frame)
    return fail(SS_ERR_UNSUPPORTED, "precision fp32 requires use_rotating_frame = 1: without the frame FP32 rounding "
                                    "accumulates past the 1e-4 bar (DESIGN.md section 5); use fp64");
  if (field_params(d.field) < 0) return fail(SS_ERR_INVALID, "field %d unknown", d.field);
  ss_sim* s = new ss_sim;
  s->d = d;
  s->dim = d.spin == SS_SPIN_HALF ? 2 : 3;
  s->P = field_params(d.field);
  s->interval = pick_interval(d);
  s->expo = pick_expo(d);
  if (!s->interval || !s->expo) {
    delete s;
    return fail(SS_ERR_UNSUPPORTED, "no kernel instance for this combination");
  }
  *out = s;
  g_err.clear();
  return SS_OK;
}

int ss_create_user(const ss_sim_desc* desc, const char* field_source, int32_t n_params, ss_sim** out) {
  if (!desc || !out || !field_source) return fail(SS_ERR_INVALID, "desc, field_source and out must be non-NULL");
  if (n_params < 1 || n_params > 64) return fail(SS_ERR_INVALID, "n_params %d outside 1..64", n_params);
  ss_sim_desc d = *desc;
  d.field = SS_FIELD_CONSTANT;      // validated like a built-in description; the field itself is the user's
  int rc = ss_create(&d, out);
  if (rc) return rc;
  ss_sim* s = *out;
  if (s->dim == 3 && d.exponentiation == SS_EXP_ANALYTIC) {
    ss_destroy(s);
    *out = nullptr;
    return fail(SS_ERR_UNSUPPORTED, "the analytic spin-one exponentiator needs omega_q == 0, which cannot be checked "
                                    "for a user field; use the Lie-Trotter exponentiator");
  }
  if ((rc = ensure_device())) { ss_destroy(s); *out = nullptr; return rc; }
  std::string err;
  if (ssb::build_user_kernel(d.spin, d.exponentiation, d.integration, d.precision == SS_FP32, field_source, n_params,
                             &s->user_kernel, &err) != 0) {
    ss_destroy(s);
    *out = nullptr;
    return fail(SS_ERR_INVALID, "%s", err.c_str());
  }
  s->user = true;
  s->P = n_params;
  s->d.field = SS_FIELD_USER;
  return SS_OK;
}

int ss_compile_user_field(const ss_sim_desc* desc, const char* field_source, int32_t n_params) {
  if (!desc || !field_source) return fail(SS_ERR_INVALID, "desc and field_source must be non-NULL");
  if (n_params < 1 || n_params > 64) return fail(SS_ERR_INVALID, "n_params %d outside 1..64", n_params);
  std::string err;
  if (ssb::build_user_kernel(desc->spin, desc->exponentiation, desc->integration, desc->precision == SS_FP32,
                             field_source, n_params, nullptr, &err) != 0)
    return fail(SS_ERR_INVALID, "%s", err.c_str());
  return SS_OK;
}

void ss_destroy(ss_sim* s) {
  if (!s) return;
  if (s->user) ssb::destroy_user_kernel(&s->user_kernel);
  for (auto& sl : s->slots)
    if (sl.buf) cudaFree(sl.buf);
  if (s->aux.buf) cudaFree(s->aux.buf);
  for (auto& st : s->streams)
    if (st) cudaStreamDestroy(st);
  for (int k = 0; k < ss_sim::kSlots; ++k) {
    if (s->computed[k]) cudaEventDestroy(s->computed[k]);
    if (s->drained[k]) cudaEventDestroy(s->drained[k]);
    if (s->stepped[k]) cudaEventDestroy(s->stepped[k]);
  }
  delete s;
}

int ss_dim(const ss_sim* s) { return s ? s->dim : fail(SS_ERR_INVALID, "sim is NULL"); }

int ss_set_split_event(ss_sim* s, void* event) {
  if (!s) return fail(SS_ERR_INVALID, "sim is NULL");
  s->split_event = static_cast<cudaEvent_t>(event);
  return SS_OK;
}

int ss_set_validation(ss_sim* s, int32_t enabled) {
  if (!s) return fail(SS_ERR_INVALID, "sim is NULL");
  s->validate = enabled ? 1 : 0;
  return SS_OK;
}

int ss_plan(double t0, double t1, double dt_int, double dt_out, int64_t* K, int64_t* L, double* dt) {
  if (!K || !L || !dt) return fail(SS_ERR_INVALID, "K, L, dt_fine must be non-NULL");
  return plan_grid(t0, t1, dt_int, dt_out, K, L, dt);
}

size_t ss_scan_workspace_bytes(int32_t dim, int64_t batch, int64_t k_count) {
  if ((dim != 2 && dim != 3) || batch < 0 || k_count < 0) return 0;
  return ssb::scan_workspace_bytes(dim, batch, k_count);
}

size_t ss_aggregate_workspace_bytes(int32_t dim, int64_t batch, int64_t k_count) {
  if ((dim != 2 && dim != 3) || batch < 0 || k_count < 0) return 0;
  return ssb::aggregate_workspace_bytes(dim, batch, k_count);
}

// Layout: [0, 256) control (validation flag) | scan workspace | fused-path run aggregates + run states (batches below
// the chain kernel's) | U (optional).
size_t ss_workspace_bytes(const ss_sim* s, int64_t batch, int64_t K, int32_t unitaries_in_workspace) {
  if (!s || batch < 0 || K < 0) return 0;
  size_t n = 256 + align256(ssb::scan_workspace_bytes(s->dim, batch, K)) + fused_bytes(s->dim, batch, K);
  if (unitaries_in_workspace) n += align256(sizeof(double) * 2 * s->dim * s->dim * (size_t)batch * (size_t)K);
  return n;
}

static int validate_inputs(ss_sim* s, int64_t batch, const double* d_sweep, const double* d_psi0, int* d_flag,
                           cudaStream_t st) {
  const int qcol = (s->dim == 3 && s->d.exponentiation == SS_EXP_ANALYTIC) ? qcol_of(s->d.field) : -1;
  cudaError_t e = cudaMemsetAsync(d_flag, 0, sizeof(int), st);
  if (e != cudaSuccess) return cuda_fail(e, "validation memset");
  e = ssb::launch_validate(batch * s->P, d_sweep, s->P, qcol, batch * 2 * s->dim, d_psi0, d_flag, st);
  if (e != cudaSuccess) return cuda_fail(e, "validation launch");
  g_launches.fetch_add(1);
  int h = 0;
  e = cudaMemcpyAsync(&h, d_flag, sizeof(int), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "validation readback");
  if (h & 1) return fail(SS_ERR_NONFINITE, "sweep parameters or state_init contain a non-finite value");
  if (h & 2) return fail(SS_ERR_INVALID, "the analytic spin-one exponentiator requires omega_q == 0 in every sweep (reading R14)");
  return SS_OK;
}

int ss_compute_unitaries(ss_sim* s, double t0, double t1, double dt_int, double dt_out, int64_t k_begin,
                         int64_t k_count, int64_t batch, const double* d_sweep, double* d_U, void* stream) {
  if (!s) return fail(SS_ERR_INVALID, "sim is NULL");
  int64_t K, L;
  double dt;
  int rc = plan_grid(t0, t1, dt_int, dt_out, &K, &L, &dt);
  if (rc) return rc;
  if (batch < 1) return fail(SS_ERR_INVALID, "batch must be >= 1");
  if (k_begin < 0 || k_count < 1 || k_begin + k_count > K)
    return fail(SS_ERR_INVALID, "interval range [%lld, %lld) outside [0, K=%lld)", (long long)k_begin,
                (long long)(k_begin + k_count), (long long)K);
  if ((rc = check_device_ptr(d_sweep, "d_sweep")) || (rc = check_device_ptr(d_U, "d_unitaries"))) return rc;
  if ((rc = ensure_device())) return rc;
  const auto p = make_params(s, t0, dt_out, dt, L, k_begin, k_count, batch, d_sweep, d_U, batch * K);
  return launch_interval_checked(s, p, static_cast<cudaStream_t>(stream));
}

int ss_scan_states(int32_t dim, int64_t batch, int64_t k_count, const double* d_U, const double* d_psi0,
                   double* d_states, void* d_ws, size_t ws_bytes, void* stream) {
  if (dim != 2 && dim != 3) return fail(SS_ERR_INVALID, "dim must be 2 or 3");
  if (batch < 1 || k_count < 1) return fail(SS_ERR_INVALID, "batch and k_count must be >= 1");
  int rc;
  if ((rc = check_device_ptr(d_U, "d_unitaries")) || (rc = check_device_ptr(d_psi0, "d_state_init")) ||
      (rc = check_device_ptr(d_states, "d_states")) || (rc = check_device_ptr(d_ws, "d_workspace")))
    return rc;
  const size_t need = ssb::scan_workspace_bytes(dim, batch, k_count);
  if (ws_bytes < need) return fail(SS_ERR_INVALID, "workspace_bytes %zu < required %zu", ws_bytes, need);
  if ((rc = ensure_device())) return rc;
  int n = 0;
  const cudaError_t e = ssb::launch_scan(dim, batch, k_count, d_U, d_psi0, d_states, d_ws,
                                         static_cast<cudaStream_t>(stream), &n);
  g_launches.fetch_add(n);
  return e == cudaSuccess ? SS_OK : cuda_fail(e, "scan launch");
}

int ss_scan_states_spin(int32_t dim, int64_t batch, int64_t k_count, const double* d_U, const double* d_psi0,
                        double* d_states, double* d_spin, void* d_ws, size_t ws_bytes, void* stream) {
  if (dim != 2 && dim != 3) return fail(SS_ERR_INVALID, "dim must be 2 or 3");
  if (batch < 1 || k_count < 1) return fail(SS_ERR_INVALID, "batch and k_count must be >= 1");
  int rc;
  if ((rc = check_device_ptr(d_U, "d_unitaries")) || (rc = check_device_ptr(d_psi0, "d_state_init")) ||
      (rc = check_device_ptr(d_ws, "d_workspace")))
    return rc;
  if (!d_states && !d_spin) return fail(SS_ERR_INVALID, "at least one of d_states, d_spin must be non-NULL");
  if (d_states && (rc = check_device_ptr(d_states, "d_states"))) return rc;
  if (d_spin && (reinterpret_cast<uintptr_t>(d_spin) & 7) != 0) return fail(SS_ERR_INVALID, "d_spin must be 8-byte aligned");
  const size_t need = ssb::scan_workspace_bytes(dim, batch, k_count);
  if (ws_bytes < need) return fail(SS_ERR_INVALID, "workspace_bytes %zu < required %zu", ws_bytes, need);
  if ((rc = ensure_device())) return rc;
  int n = 0;
  const cudaError_t e = ssb::launch_scan(dim, batch, k_count, d_U, d_psi0, d_states, d_ws,
                                         static_cast<cudaStream_t>(stream), &n, d_spin);
  g_launches.fetch_add(n);
  return e == cudaSuccess ? SS_OK : cuda_fail(e, "scan launch");
}

int ss_scan_states_su2(int32_t dim, int64_t batch, int64_t k_count, const double* d_ops, const double* d_psi0,
                       double* d_states, double* d_spin, void* d_ws, size_t ws_bytes, void* stream) {
  if (dim != 2 && dim != 3) return fail(SS_ERR_INVALID, "dim must be 2 or 3");
  if (batch < 1 || k_count < 1) return fail(SS_ERR_INVALID, "batch and k_count must be >= 1");
  int rc;
  if ((rc = check_device_ptr(d_ops, "d_ops")) || (rc = check_device_ptr(d_psi0, "d_state_init")) ||
      (rc = check_device_ptr(d_ws, "d_workspace")))
    return rc;
  if (!d_states && !d_spin) return fail(SS_ERR_INVALID, "at least one of d_states, d_spin must be non-NULL");
  if (d_states && (rc = check_device_ptr(d_states, "d_states"))) return rc;
  if (d_spin && (reinterpret_cast<uintptr_t>(d_spin) & 7) != 0) return fail(SS_ERR_INVALID, "d_spin must be 8-byte aligned");
  const size_t need = ssb::scan_workspace_bytes(dim, batch, k_count);
  if (ws_bytes < need) return fail(SS_ERR_INVALID, "workspace_bytes %zu < required %zu", ws_bytes, need);
  if ((rc = ensure_device())) return rc;
  int n = 0;
  const cudaError_t e = ssb::launch_scan(dim, batch, k_count, d_ops, d_psi0, d_states, d_ws,
                                         static_cast<cudaStream_t>(stream), &n, d_spin, ssb::OP_SU2);
  g_launches.fetch_add(n);
  return e == cudaSuccess ? SS_OK : cuda_fail(e, "scan launch");
}

int ss_chain_aggregate(int32_t dim, int64_t batch, int64_t k_count, const double* d_U, double* d_agg, void* d_ws,
                       size_t ws_bytes, void* stream) {
  if (dim != 2 && dim != 3) return fail(SS_ERR_INVALID, "dim must be 2 or 3");
  if (batch < 1 || k_count < 1) return fail(SS_ERR_INVALID, "batch and k_count must be >= 1");
  int rc;
  if ((rc = check_device_ptr(d_U, "d_unitaries")) || (rc = check_device_ptr(d_agg, "d_aggregate")) ||
      (rc = check_device_ptr(d_ws, "d_workspace")))
    return rc;
  const size_t need = ssb::aggregate_workspace_bytes(dim, batch, k_count);
  if (ws_bytes < need) return fail(SS_ERR_INVALID, "workspace_bytes %zu < required %zu", ws_bytes, need);
  if ((rc = ensure_device())) return rc;
  int n = 0;
  const cudaError_t e = ssb::launch_aggregate(dim, batch, k_count, d_U, d_agg, d_ws, static_cast<cudaStream_t>(stream), &n);
  g_launches.fetch_add(n);
  return e == cudaSuccess ? SS_OK : cuda_fail(e, "aggregate launch");
}

int ss_compose_carry(int32_t dim, int64_t batch, int32_t n_parts, int32_t part, const double* d_aggs,
                     const double* d_psi0, double* d_carry, void* stream) {
  if (dim != 2 && dim != 3) return fail(SS_ERR_INVALID, "dim must be 2 or 3");
  if (batch < 1) return fail(SS_ERR_INVALID, "batch must be >= 1");
  if (n_parts < 1 || part < 0 || part >= n_parts) return fail(SS_ERR_INVALID, "part %d outside [0, %d)", part, n_parts);
  int rc;
  if ((part > 0 && (rc = check_device_ptr(d_aggs, "d_aggregates"))) || (rc = check_device_ptr(d_psi0, "d_state_init")) ||
      (rc = check_device_ptr(d_carry, "d_carry")))
    return rc;
  if ((rc = ensure_device())) return rc;
  const cudaError_t e = ssb::launch_compose_carry(dim, batch, part, d_aggs, d_psi0, d_carry, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "compose_carry launch");
  g_launches.fetch_add(1);
  return SS_OK;
}

int ss_evaluate(ss_sim* s, double t0, double t1, double dt_int, double dt_out, int64_t batch, const double* d_sweep,
                const double* d_psi0, double* d_states, double* d_U, void* d_ws, size_t ws_bytes, void* stream) {
  if (!s) return fail(SS_ERR_INVALID, "sim is NULL");
  int64_t K, L;
  double dt;
  int rc = plan_grid(t0, t1, dt_int, dt_out, &K, &L, &dt);
  if (rc) return rc;
  if (batch < 1) return fail(SS_ERR_INVALID, "batch must be >= 1");
  if ((rc = check_device_ptr(d_sweep, "d_sweep")) || (rc = check_device_ptr(d_psi0, "d_state_init")) ||
      (rc = check_device_ptr(d_states, "d_states")) || (rc = check_device_ptr(d_ws, "d_workspace")))
    return rc;
  if ((reinterpret_cast<uintptr_t>(d_ws) & 255) != 0) return fail(SS_ERR_INVALID, "d_workspace must be 256-byte aligned");
  const size_t need = ss_workspace_bytes(s, batch, K, d_U == nullptr);
  if (ws_bytes < need) return fail(SS_ERR_INVALID, "workspace_bytes %zu < required %zu", ws_bytes, need);
  if ((rc = ensure_device())) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* w = static_cast<char*>(d_ws);
  void* scan_ws = w + 256;
  double* U = d_U ? d_U
                  : reinterpret_cast<double*>(w + 256 + align256(ssb::scan_workspace_bytes(s->dim, batch, K)) +
                                              fused_bytes(s->dim, batch, K));
  if (s->validate && (rc = validate_inputs(s, batch, d_sweep, d_psi0, reinterpret_cast<int*>(w), st))) return rc;
  auto p = make_params(s, t0, dt_out, dt, L, 0, K, batch, d_sweep, U, batch * K);
  // U_k only feeds the scan: SU(2)-form paths pass it compact (the workspace is sized for the dense layout)
  if (!d_U && su2_form(s)) p.op_format = ssb::OP_SU2;
  char* fw = w + 256 + align256(ssb::scan_workspace_bytes(s->dim, batch, K));   // fused region
  return launch_path(s, p, d_psi0, d_states, scan_ws, fused_batch(batch) ? fw : nullptr, st, st, nullptr);
}

int ss_exponentiate(const ss_sim* s, int64_t n, const double* d_args, double* d_out, void* stream) {
  if (!s) return fail(SS_ERR_INVALID, "sim is NULL");
  if (n < 1) return fail(SS_ERR_INVALID, "n must be >= 1");
  int rc;
  if ((rc = check_device_ptr(d_args, "d_args")) || (rc = check_device_ptr(d_out, "d_out"))) return rc;
  if ((rc = ensure_device())) return rc;
  const cudaError_t e = s->expo(n, d_args, s->d.trotter_cutoff, d_out, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "exponentiate launch");
  g_launches.fetch_add(1);
  return SS_OK;
}

int ss_magnus_bound(ss_sim* s, double t0, double t1, double dt_int, double dt_out, int64_t batch,
                    const double* d_sweep, double* d_out, void* stream) {
  if (!s) return fail(SS_ERR_INVALID, "sim is NULL");
  int64_t K, L;
  double dt;
  int rc = plan_grid(t0, t1, dt_int, dt_out, &K, &L, &dt);
  if (rc) return rc;
  if (batch < 1) return fail(SS_ERR_INVALID, "batch must be >= 1");
  if ((rc = check_device_ptr(d_sweep, "d_sweep"))) return rc;
  if (!d_out || (reinterpret_cast<uintptr_t>(d_out) & 7) != 0) return fail(SS_ERR_INVALID, "d_out must be 8-byte aligned");
  if ((rc = ensure_device())) return rc;
  const ssb::MagnusLaunchFn fn = s->user ? nullptr : pick_magnus(s->d);
  if (!s->user && !fn) return fail(SS_ERR_UNSUPPORTED, "no Magnus diagnostic instance for this combination");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemsetAsync(d_out, 0, sizeof(double) * (size_t)batch, st);
  if (e != cudaSuccess) return cuda_fail(e, "magnus memset");
  const auto p = make_params(s, t0, dt_out, dt, L, 0, K, batch, d_sweep, nullptr, batch * K);
  e = s->user ? ssb::launch_user_magnus(s->user_kernel, p, d_out, st) : fn(p, d_out, st);
  if (e != cudaSuccess) return cuda_fail(e, "magnus launch");
  g_launches.fetch_add(1);
  return SS_OK;
}

int ss_spin_projection(int32_t spin, int64_t n, const double* d_states, double* d_out, void* stream) {
  if (spin != SS_SPIN_HALF && spin != SS_SPIN_ONE) return fail(SS_ERR_INVALID, "spin must be 1 or 2");
  if (n < 1) return fail(SS_ERR_INVALID, "n must be >= 1");
  int rc;
  if ((rc = check_device_ptr(d_states, "d_states")) || (rc = check_device_ptr(d_out, "d_out"))) return rc;
  if ((rc = ensure_device())) return rc;
  const cudaError_t e = ssb::launch_spin_projection(spin == SS_SPIN_HALF ? 2 : 3, n, d_states, d_out,
                                                    static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "spin_projection launch");
  g_launches.fetch_add(1);
  return SS_OK;
}

// Host-buffer pipeline plan (ss_evaluate_host, ss_host_chunk_plan): pure host logic, no device calls beyond the SM
// count.  kind 0: batch chunks of geometrically shrinking size (sizes = sweeps); kind 1: tent-shaped time chunks,
// kind 2: the wave-aligned time pair (sizes = intervals).
//
// Time chunks: large batches (the chain scan is sequential per sweep — bit-identical to ss_evaluate), and long
// sweeps of small batches whose interval work spans ≥ 6 waves per chunk on average (one sweep of 1e6 intervals,
// C4); there the single-sweep scan restarts from the carry each chunk, so states agree with ss_evaluate to
// rounding (a different product order), not bit for bit.
#ifndef SS_HOST_SCAN_STREAM
#define SS_HOST_SCAN_STREAM 1   // 0: time chunks scan on the compute stream (comparison builds)
#endif
static int plan_host_chunks(const ss_sim* s, int64_t K, int64_t L, int64_t batch, int32_t n_chunks, int32_t* kind,
                     std::vector<int64_t>& ks) {
  ks.clear();
  const bool big_batch = batch >= ssb::chain_min_batch();
  const double waves = (double)batch * K * choose_split(s, batch * K, L) / resident_threads(s);
  const bool single = n_chunks == 1;                       // the caller asked for one chunk
  if (n_chunks <= 0) {        // auto: ≈ 40 time chunks where they apply (measured best for C3: e2e 0.97 of device),
    int64_t tc = std::min<int64_t>(40, K / 4);            // else 4 geometric batch chunks
    if (!big_batch) tc = std::min<int64_t>(tc, (int64_t)(waves / 8.0));   // C4: 6 (measured best)
    n_chunks = tc >= 6 ? (int32_t)tc : 4;
  }
  const bool tent = n_chunks >= 6 && K >= 4 * (int64_t)n_chunks && (big_batch || waves >= 6.0 * n_chunks);
  // Wave-aligned pair (C2: one sweep of 1e5 intervals = 2.6 waves, too short for the tent): chunk A holds the whole
  // waves but the last, chunk B the rest.  Interval work still takes ⌈waves⌉ wave-times in total, and the D2H of
  // chunk A (most of the states) overlaps chunk B's kernels; only chunk B's copy is left exposed.
  const int64_t wave_iv = (int64_t)(resident_threads(s) / choose_split(s, batch * K, L)) / batch;   // intervals/wave
  const int64_t pair_waves = (int64_t)std::ceil(waves) - 1;
  const bool pair = !tent && !single && !big_batch && batch <= 4 && waves >= 1.2 && wave_iv >= 1 && pair_waves >= 1 &&
                    pair_waves * wave_iv < K;
  if (pair) {
    *kind = 2;
    ks = {pair_waves * wave_iv, K - pair_waves * wave_iv};
    return SS_OK;
  }
  if (tent) {
    // Tent-shaped sizes — small first chunks so the device→host copies start early, small last ones so little copy
    // is left exposed — with weights 1, 2, 3, …, 3, 1, ½, ¼, ¼ (three staging slots: the copy of chunk c overlaps
    // chunks c+1 and c+2); boundaries from the cumulative weights (rounding errors do not accumulate), every chunk
    // ≥ 1 interval.
    *kind = 1;
    std::vector<double> w = {1.0, 2.0};
    while ((int)w.size() < n_chunks - 4) w.push_back(3.0);
    for (double x : {1.0, 0.5, 0.25, 0.25}) w.push_back(x);
    double wsum = 0;
    for (double x : w) wsum += x;
    const int64_t nc = (int64_t)w.size();
    double cum = 0.0;
    int64_t b = 0;
    for (int64_t c = 0; c < nc; ++c) {
      cum += w[c];
      int64_t nb = (c + 1 == nc) ? K : (int64_t)std::llround(K * cum / wsum);
      nb = std::min(std::max(nb, b + 1), K - (nc - c - 1));
      ks.push_back(nb - b);
      b = nb;
    }
    return SS_OK;
  }
  // Geometric batch chunks (B/2, B/4, …, the last two equal): early chunks are big (full-speed chain scan, long
  // compute that hides the previous chunk's D2H), the final chunk — whose D2H cannot be hidden — is small.
  *kind = 0;
  if (n_chunks > batch) n_chunks = (int32_t)batch;
  int64_t left = batch;
  for (int c = 0; c < n_chunks && left > 0; ++c) {
    const int64_t cb = (c == n_chunks - 1) ? left : std::max<int64_t>(1, (left + 1) / 2);
    ks.push_back(cb);
    left -= cb;
  }
  return SS_OK;
}

int ss_evaluate_host(ss_sim* s, double t0, double t1, double dt_int, double dt_out, int64_t batch, const double* h_sweep,
                     const double* h_psi0, double* h_states, double* h_U, int32_t n_chunks) {
  if (!s) return fail(SS_ERR_INVALID, "sim is NULL");
  int64_t K, L;
  double dt;
  int rc = plan_grid(t0, t1, dt_int, dt_out, &K, &L, &dt);
  if (rc) return rc;
  if (batch < 1) return fail(SS_ERR_INVALID, "batch must be >= 1");
  if (!h_sweep || !h_psi0 || !h_states) return fail(SS_ERR_INVALID, "h_sweep, h_state_init, h_states must be non-NULL");
  // host-side input validation (host data: no device round trip needed)
  const int qcol = (s->dim == 3 && s->d.exponentiation == SS_EXP_ANALYTIC) ? qcol_of(s->d.field) : -1;
  for (int64_t i = 0; i < batch * s->P; ++i) {
    if (!std::isfinite(h_sweep[i])) return fail(SS_ERR_NONFINITE, "sweep parameter %lld is not finite", (long long)i);
    if (qcol >= 0 && i % s->P == qcol && h_sweep[i] != 0.0)
      return fail(SS_ERR_INVALID, "the analytic spin-one exponentiator requires omega_q == 0 in every sweep (reading R14)");
  }
  for (int64_t i = 0; i < batch * 2 * s->dim; ++i)
    if (!std::isfinite(h_psi0[i])) return fail(SS_ERR_NONFINITE, "state_init value %lld is not finite", (long long)i);
  if ((rc = ensure_device())) return rc;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  if (s->device != dev) {  // (re)create per-device streams/events and drop buffers of another device
    for (auto& st : s->streams) if (st) cudaStreamDestroy(st), st = nullptr;
    for (auto& sl : s->slots) if (sl.buf) cudaFree(sl.buf), sl.buf = nullptr, sl.cap = 0;
    if (s->aux.buf) cudaFree(s->aux.buf), s->aux.buf = nullptr, s->aux.cap = 0;
    for (int k = 0; k < ss_sim::kSlots; ++k) {
      if (s->computed[k]) cudaEventDestroy(s->computed[k]), s->computed[k] = nullptr;
      if (s->drained[k]) cudaEventDestroy(s->drained[k]), s->drained[k] = nullptr;
      if (s->stepped[k]) cudaEventDestroy(s->stepped[k]), s->stepped[k] = nullptr;
    }
    for (auto& st : s->streams)
      if ((e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking)) != cudaSuccess) return cuda_fail(e, "stream create");
    for (int k = 0; k < ss_sim::kSlots; ++k)
      if ((e = cudaEventCreateWithFlags(&s->computed[k], cudaEventDisableTiming)) != cudaSuccess ||
          (e = cudaEventCreateWithFlags(&s->drained[k], cudaEventDisableTiming)) != cudaSuccess ||
          (e = cudaEventCreateWithFlags(&s->stepped[k], cudaEventDisableTiming)) != cudaSuccess)
        return cuda_fail(e, "event create");
    s->device = dev;
  }
  const int D = s->dim;
  // Synchronous call: on every return — including an error after work was enqueued — all three streams are drained
  // first, so no copy into the caller's host buffers or scan over the carry is still in flight.
  struct DrainOnExit {
    cudaStream_t* st;
    ~DrainOnExit() {
      for (int k = 0; k < 3; ++k)
        if (st[k]) (void)cudaStreamSynchronize(st[k]);
    }
  } drain{s->streams};
  auto ensure = [&](ss_sim::Slot& sl, size_t bytes) -> cudaError_t {
    if (sl.cap >= bytes) return cudaSuccess;
    if (sl.buf) cudaFree(sl.buf);
    sl.buf = nullptr;
    sl.cap = 0;
    const cudaError_t r = cudaMalloc(&sl.buf, bytes);
    if (r == cudaSuccess) sl.cap = bytes;
    return r;
  };
  cudaStream_t cs = s->streams[0], xs = s->streams[1];

  int32_t kind = 0;
  std::vector<int64_t> ks;
  plan_host_chunks(s, K, L, batch, n_chunks, &kind, ks);
  // Scans on their own stream only for the tent over few sweeps (C4: the single-sweep scan of chunk c beside chunk
  // c+1's interval kernel, e2e 0.957 → 0.970 of the device rate).  Measured worse elsewhere: the chain kernel of
  // large batches (C3: 0.97 → 0.80) and the pair's cooperative scan (C2: 0.71 → 0.65) then wait for the next
  // interval kernel's blocks to drain, which delays the copies.
  cudaStream_t ss = (SS_HOST_SCAN_STREAM && kind == 1 && batch < ssb::chain_min_batch()) ? s->streams[2] : cs;
  if (kind != 0) {
    // Chunk the TIME axis, all sweeps per chunk (for large batches the per-sweep chain kernel stays at full width and
    // is sequential per sweep, so the states are bit-identical to one ss_evaluate).  Chunk c = intervals [k0, k0 + kc)
    // of every sweep, started from the running carry (the previous chunk's last states).
    int64_t kc_max = 0;
    for (int64_t x : ks) kc_max = std::max(kc_max, x);
    const size_t sweep_b = align256(sizeof(double) * s->P * batch), carry_b = align256(sizeof(double) * 2 * D * batch);
    const size_t states_b = align256(sizeof(double) * 2 * D * (size_t)batch * (kc_max + 1));
    const size_t U_b = align256(sizeof(double) * 2 * D * D * (size_t)batch * kc_max);
    const size_t scan_b = align256(ssb::scan_workspace_bytes(D, batch, kc_max));
    const size_t fused_b = fused_bytes(D, batch, kc_max);
    if ((e = ensure(s->aux, sweep_b + carry_b)) != cudaSuccess) return cuda_fail(e, "cudaMalloc (host-API staging)");
    for (int k = 0; k < ss_sim::kSlots; ++k)
      if ((e = ensure(s->slots[k], states_b + U_b + scan_b + fused_b)) != cudaSuccess)
        return cuda_fail(e, "cudaMalloc (host-API staging)");
    double* d_sweep = static_cast<double*>(s->aux.buf);
    double* d_carry = reinterpret_cast<double*>(static_cast<char*>(s->aux.buf) + sweep_b);
    if ((e = cudaMemcpyAsync(d_sweep, h_sweep, sizeof(double) * s->P * batch, cudaMemcpyHostToDevice, cs)) ||
        (e = cudaMemcpyAsync(d_carry, h_psi0, sizeof(double) * 2 * D * batch, cudaMemcpyHostToDevice, cs)))
      return cuda_fail(e, "H2D copy");
    const size_t row = sizeof(double) * 2 * D;                   // one state
    for (size_t c = 0, k0 = 0; c < ks.size(); k0 += ks[c], ++c) {
      const int64_t kc = ks[c];
      const int k = (int)(c % ss_sim::kSlots);
      char* base = static_cast<char*>(s->slots[k].buf);
      double* d_states = reinterpret_cast<double*>(base);
      double* d_U = reinterpret_cast<double*>(base + states_b);
      void* d_scan = base + states_b + U_b;
      // [cs] interval kernel of chunk c (its slot's D2H, three chunks back, must have drained) → stepped[k];
      // [ss] scan of chunk c from the running carry, carry ← its last states → computed[k] (the scans stay in chunk
      // order on ss, so the carry chain is sequential; chunk c+1's interval kernel runs beside chunk c's scan).
      if (c >= (size_t)ss_sim::kSlots && (e = cudaStreamWaitEvent(cs, s->drained[k], 0)) != cudaSuccess)
        return cuda_fail(e, "event wait");
      auto p = make_params(s, t0, dt_out, dt, L, (int64_t)k0, kc, batch, d_sweep, d_U, batch * K);
      if (!h_U && su2_form(s)) p.op_format = ssb::OP_SU2;
      if ((rc = launch_path(s, p, d_carry, d_states, d_scan, fused_b ? base + states_b + U_b + scan_b : nullptr, cs, ss,
                            s->stepped[k])))
        return rc;
      // carry ← states[:, kc]
      if ((e = copy_rows(d_carry, row, d_states + (size_t)kc * 2 * D, row * (kc + 1), row, batch,
                                 cudaMemcpyDeviceToDevice, ss)))
        return cuda_fail(e, "carry copy");
      if ((e = cudaEventRecord(s->computed[k], ss)) || (e = cudaStreamWaitEvent(xs, s->computed[k], 0)))
        return cuda_fail(e, "event record/wait");
      const size_t first = (c == 0) ? 0 : 1;                     // states[:, 0] of chunk c > 0 is the carry
      if ((e = copy_rows(h_states + (k0 + first) * 2 * D, row * (K + 1), d_states + first * 2 * D,
                                 row * (kc + 1), row * (kc + 1 - first), batch, cudaMemcpyDeviceToHost, xs)))
        return cuda_fail(e, "D2H copy (states)");
      if (h_U && (e = copy_rows(h_U + k0 * 2 * D * D, row * D * K, d_U, row * D * kc, row * D * kc, batch,
                                        cudaMemcpyDeviceToHost, xs)))
        return cuda_fail(e, "D2H copy (unitaries)");
      if ((e = cudaEventRecord(s->drained[k], xs))) return cuda_fail(e, "event record");
    }
    for (int k = 0; k < 3; ++k)
      if ((e = cudaStreamSynchronize(s->streams[k])) != cudaSuccess) return cuda_fail(e, "stream synchronize");
    return SS_OK;
  }
  // Geometric batch chunks (plan_host_chunks, kind 0).
  const std::vector<int64_t>& sizes = ks;
  n_chunks = (int32_t)sizes.size();
  const int64_t cb_max = sizes[0];
  const size_t sweep_b = align256(sizeof(double) * s->P * cb_max);
  const size_t psi0_b = align256(sizeof(double) * 2 * D * cb_max);
  const size_t states_b = align256(sizeof(double) * 2 * D * (size_t)cb_max * (K + 1));
  const size_t U_b = align256(sizeof(double) * 2 * D * D * (size_t)cb_max * K);
  const size_t scan_b = align256(ssb::scan_workspace_bytes(D, cb_max, K));
  const size_t fused_b = fused_bytes(D, cb_max, K);   // a chunk has ≤ cb_max sweeps: fused_bytes(D, cb, K) ≤ fused_b
  const size_t slot_bytes = sweep_b + psi0_b + states_b + U_b + scan_b + fused_b;
  const int nslots = n_chunks > 1 ? 2 : 1;
  for (int k = 0; k < nslots; ++k)
    if ((e = ensure(s->slots[k], slot_bytes)) != cudaSuccess) return cuda_fail(e, "cudaMalloc (host-API staging)");
  // Chunk c: [compute stream] wait drained[slot] (its D2H two chunks ago) → H2D inputs → kernels → record
  // computed[slot];  [copy stream] wait computed[slot] → D2H → record drained[slot].  Compute stays serial over
  // chunks (each chunk fills the GPU), so the D2H of chunk c overlaps the kernels of chunk c+1.
  for (int64_t c = 0, b0 = 0; c < n_chunks; ++c) {
    const int64_t cb = sizes[c];
    if (cb <= 0) break;
    const int k = (int)(c % nslots);
    char* base = static_cast<char*>(s->slots[k].buf);
    double* d_sweep = reinterpret_cast<double*>(base);
    double* d_psi0 = reinterpret_cast<double*>(base + sweep_b);
    double* d_states = reinterpret_cast<double*>(base + sweep_b + psi0_b);
    double* d_U = reinterpret_cast<double*>(base + sweep_b + psi0_b + states_b);
    void* d_scan = base + sweep_b + psi0_b + states_b + U_b;
    if (c >= nslots && (e = cudaStreamWaitEvent(cs, s->drained[k], 0)) != cudaSuccess) return cuda_fail(e, "event wait");
    if ((e = cudaMemcpyAsync(d_sweep, h_sweep + b0 * s->P, sizeof(double) * s->P * cb, cudaMemcpyHostToDevice, cs)) ||
        (e = cudaMemcpyAsync(d_psi0, h_psi0 + b0 * 2 * D, sizeof(double) * 2 * D * cb, cudaMemcpyHostToDevice, cs)))
      return cuda_fail(e, "H2D copy");
    auto p = make_params(s, t0, dt_out, dt, L, 0, K, cb, d_sweep, d_U, batch * K);   // S of the whole batch
    if (!h_U && su2_form(s)) p.op_format = ssb::OP_SU2;
    char* d_fused = static_cast<char*>(d_scan) + scan_b;
    if ((rc = launch_path(s, p, d_psi0, d_states, d_scan, fused_b && fused_batch(cb) ? d_fused : nullptr, cs, cs,
                          nullptr)))
      return rc;
    if ((e = cudaEventRecord(s->computed[k], cs)) || (e = cudaStreamWaitEvent(xs, s->computed[k], 0)))
      return cuda_fail(e, "event record/wait");
    if ((e = cudaMemcpyAsync(h_states + b0 * 2 * D * (K + 1), d_states, sizeof(double) * 2 * D * cb * (K + 1),
                             cudaMemcpyDeviceToHost, xs)))
      return cuda_fail(e, "D2H copy (states)");
    if (h_U && (e = cudaMemcpyAsync(h_U + b0 * 2 * D * D * K, d_U, sizeof(double) * 2 * D * D * cb * K,
                                    cudaMemcpyDeviceToHost, xs)))
      return cuda_fail(e, "D2H copy (unitaries)");
    if ((e = cudaEventRecord(s->drained[k], xs))) return cuda_fail(e, "event record");
    b0 += cb;
  }
  for (int k = 0; k < 2; ++k)
    if ((e = cudaStreamSynchronize(s->streams[k])) != cudaSuccess) return cuda_fail(e, "stream synchronize");
  return SS_OK;
}

int ss_host_chunk_plan(const ss_sim* s, double t0, double t1, double dt_int, double dt_out, int64_t batch,
                       int32_t n_chunks, int32_t* kind, int64_t* sizes, int32_t cap, int32_t* count) {
  if (!s) return fail(SS_ERR_INVALID, "sim is NULL");
  if (!kind || !count || (cap > 0 && !sizes)) return fail(SS_ERR_INVALID, "kind, count (and sizes) must be non-NULL");
  int64_t K, L;
  double dt;
  int rc = plan_grid(t0, t1, dt_int, dt_out, &K, &L, &dt);
  if (rc) return rc;
  if (batch < 1) return fail(SS_ERR_INVALID, "batch must be >= 1");
  std::vector<int64_t> ks;
  plan_host_chunks(s, K, L, batch, n_chunks, kind, ks);
  *count = (int32_t)ks.size();
  if ((int64_t)ks.size() > (int64_t)cap) return fail(SS_ERR_INVALID, "cap (%d) < number of chunks (%d)", cap, *count);
  for (size_t c = 0; c < ks.size(); ++c) sizes[c] = ks[c];
  return SS_OK;
}

}  // extern "C"
