#!/usr/bin/env python
"""bench.py — fine steps/s of the Spinsim hot path on B200 (BASELINE.json metric), one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C3|C2|C5|C4|G1] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...           (the driver's launch for N > 1)

A "step" is one pass of the whole hot path (SURVEY §8(a) rows a1–a9: interval kernel + state scan) over one batch.
Default workload: C3 (BASELINE configs[2]) — 8192 spin-one sweeps × 10 ms, δt = 100 ns, Δt = 1 µs, Lie–Trotter
τ = 24, rotating frame — the batch-summed FP64 workload the metric is quoted on "at 1/2/4/8 B200".  Multi-GPU
shards sweeps (no data-path collective); `--scaling strong` (default: BASELINE configs[2], "8192 … sharded across
1/2/4/8 GPUs") splits the 8192 sweeps into contiguous blocks, one per rank; `--scaling weak` keeps 8192 sweeps per
rank.  `--emulate-ranks N` (one GPU, no torchrun) times rank 0's shard of an N-rank strong-scaling run and adds the
predicted N-GPU value (shard rate × N: sweep sharding has no exchange) — the per-rank shard shapes of the SCALE run.  Timing: CUDA events on the launching stream, barrier + synchronize on both sides, max
over ranks (all_reduce MAX).  Working set (U 11.8 GB + states 3.9 GB per rank) ≫ L2 (126 MB), so no flush is needed.

`--impl reference` times the CPU oracle (oracle/, the "reference arm" of this tier) on the host cores on a bounded
sample of the same workload; under torchrun only rank 0 runs it.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
UNIT = "fine steps/s"
# Nominal FP64 peak: 148 SMs × 64 FP64 FMA/clk/SM × 2 flop × 1.965 GHz (max SM clock).
N_SM, FP64_FMA_PER_CLK_SM, SM_MAX_MHZ = 148, 64, 1965.0
FP64_PEAK_TFLOPS = N_SM * FP64_FMA_PER_CLK_SM * 2 * SM_MAX_MHZ * 1e6 / 1e12
# FP32 mode: 128 FP32 FMA/clk/SM (2:1 FP32:FP64 on B200, confirmed by ncu's roofline note), same clock.
FP32_PEAK_TFLOPS = 2 * FP64_PEAK_TFLOPS


def algorithmic_flops_per_fine_step(spin: str, expo: str, tau: int, method: str = "cf4") -> int:
    """Arithmetic of one fine step in this implementation's formulation, counting every real +, −, ×
    once (an FMA is 2).

    spin-one Lie–Trotter: residual squaring of the complex-symmetric unitary leapfrog factor T₀ in scaled double-angle
    form (x̃' = −ỹ², ỹ' = (x̃ + 2I)ỹ on its 6 unique entries, DESIGN.md §5 item 13) = 63 flop (39 FP64 instructions)
    × τ per exponential, residual product b + a(I + b) = 219 (3×3) per exponential; field, frame, T − I construction
    and phases are not counted (a lower bound; ncu's executed count is in profiles/r01/).
    spin-half: per CF4 step 2 × (SU(2) closed form + SU(2)-parametrised residual product 36) plus the weights, field
    samples, frame rotation, phase steppers and grid — 163 in total, the ncu-executed count on C4 (2·DFMA + DMUL +
    DADD per step: 61.1 DFMA + 32.3 DMUL + 8.1 DADD, profiles/r01/s8_final/flops_c4.csv, after DESIGN.md §5 items
    10, 12, 15 and the folded weights).  Steps with r > 2^-13 (longer series, e.g. C5 at 100 ns) execute ≈ 26 more,
    so their reported fraction is a lower bound.
    general spin-one (lie_trotter_su3, readings R19/R20): the same 63-flop symmetric squaring × τ on the
    tridiagonalised factor T₀, the conjugation W (T₀^n − I) W† = 24 complex multiply-adds = 192 flop, residual product
    219; the tridiagonalisation and T₀ construction are not counted.
    spin-one analytic (reading R14): accumulated in SU(2) form and mapped by D¹ once per interval (DESIGN.md §5
    item 11), so its fine step is the spin-half step: 163."""
    n_exp = 2 if method == "cf4" else 1
    if spin == "one" and expo == "analytic":
        spin = "half"
    if spin == "one":
        prod = 219
        per_exp = {"lie_trotter": 63 * tau, "lie_trotter_su3": 63 * tau + 192}.get(expo, 0)
        return n_exp * (per_exp + prod)
    return 163 if method == "cf4" else 82


def dense_equivalent_flops_per_fine_step(spin: str, expo: str, tau: int, method: str = "cf4") -> int:
    """SURVEY §8(d)'s per-unit figure: the same step with dense 3×3 squarings as written in P:462, (a + 2I)a =
    201 flop each (context only)."""
    n_exp = 2 if method == "cf4" else 1
    if spin == "one":
        return n_exp * ((201 * tau if expo in ("lie_trotter", "lie_trotter_su3") else 0) + 234)
    return n_exp * 72


def ncu_traffic(kernel: str, workload: str, full_size: bool):
    """DRAM bytes per launch of this kernel on this workload from the committed ncu capture (profiles/), or None."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
    except (OSError, ValueError):
        return None
    e = d.get(f"{kernel}@{workload}") if full_size else None
    return e["bytes"] if e else None


def executed_flops(kernel: str, workload: str):
    """FP64 flops one fine step EXECUTES (ncu SASS op counts: 2·DFMA + DMUL + DADD per fine step) for this kernel on
    this workload, from the committed capture (profiles/executed_flops.json), or None."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "executed_flops.json")))
    except (OSError, ValueError):
        return None
    return d.get(f"{kernel}@{workload}")


def executed_of(kernel: str, workload: str, fine_steps: int, ms: float, peak: float):
    e = executed_flops(kernel, workload)
    if not e:
        return None
    tf = e["flops_per_fine_step"] * fine_steps / (ms * 1e-3) / 1e12
    return {"flops_per_fine_step": e["flops_per_fine_step"], "achieved": tf, "frac": tf / peak, "source": e["source"]}


def hbm_peak_gbs():
    """HBM roofline denominator: MEASURED_PEAKS.json's STREAM-style copy (driver-written), else the profiling guide's
    fallback 6.65 TB/s (B200_PROFILING.md) — returned with which one it is."""
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        v = float(d["hbm_gbs"])
        if v > 0:
            return v, "of measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, ValueError, KeyError, TypeError):
        pass
    return 6650.0, "of fallback (B200_PROFILING.md: 6.65 TB/s)"


def scan_bytes_per_interval(dim: int, compact: bool = False) -> int:
    """Algorithmic bytes of the state scan per interval: read U_k (dense dim×dim complex128, or the 32-B SU(2)
    element the SU(2)-form paths hand over when U_k is not an output) + write ψ_{k+1}."""
    return (2 * (2 if compact else dim * dim) + 2 * dim) * 8


def su2_form(w) -> bool:
    """spin-half and analytic spin-one accumulate in SU(2) (DESIGN.md §5 items 10-11): compact operators."""
    return w.spin == "half" or w.expo == "analytic"


def get_workload(name: str, batch: int, expo: str | None = None) -> W.Workload:
    if name == "C3":
        return W.c3_batched(batch=batch)
    if name == "C2":
        return W.c2_neural(dt_int=100e-9)
    if name == "C5":
        return W.c5_matrix(expo or "lie_trotter", batch=100)
    if name == "C4":
        return W.c4_long()
    if name == "G1":
        return W.g1_su3(batch=batch)
    raise ValueError(name)


def _nvml_handle(index: int):
    """NVML handle of CUDA device `index` (by UUID, so CUDA_VISIBLE_DEVICES remapping is respected), or None."""
    try:
        import pynvml
        import torch
        pynvml.nvmlInit()
        try:
            return pynvml.nvmlDeviceGetHandleByUUID("GPU-" + str(torch.cuda.get_device_properties(index).uuid))
        except Exception:
            return pynvml.nvmlDeviceGetHandleByIndex(index)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region, plus NVML polled every 2 ms
    by a host thread (so sub-second regions such as C2's and C4's also carry clock samples)."""
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def _poll_nvml(self):
        import pynvml
        R = pynvml
        bits = {"hw_slowdown": R.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": R.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": R.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": R.nvmlClocksEventReasonSwPowerCap}
        while not self.stop.is_set():
            try:
                sm = R.nvmlDeviceGetClockInfo(self.h, R.NVML_CLOCK_SM)
                mx = R.nvmlDeviceGetMaxClockInfo(self.h, R.NVML_CLOCK_SM)
                pw = R.nvmlDeviceGetPowerUsage(self.h) / 1000.0
                rs = R.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.nvml.append((float(sm), float(mx), pw, sorted(n for n, b in bits.items() if rs & b)))
            except Exception:
                return
            self.stop.wait(0.002)

    def __enter__(self):
        self.nvml = []
        self.stop = threading.Event()
        self.h = _nvml_handle(self.index)
        if self.h is not None:
            self.nvml_thread = threading.Thread(target=self._poll_nvml, daemon=True)
            self.nvml_thread.start()
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.QUERY}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        self.stop.set()
        if self.h is not None:
            self.nvml_thread.join(timeout=1)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, power, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
                power.append(float(f[3]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        n_smi = len(sm)
        for (a, b, c, r) in self.nvml:
            sm.append(a)
            mx.append(b)
            power.append(c)
            reasons.update(r)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm), "samples_nvidia_smi": n_smi, "samples_nvml": len(self.nvml),
                "power_w_median": float(np.median(power))}


BAD_REASONS = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}


def clocks_ok(c: dict) -> bool:
    """Timing rule: no hardware/thermal slowdown, and SM clock not stuck well below max without a reason."""
    if set(c.get("reasons", [])) & BAD_REASONS:
        return False
    if c.get("sm_mhz") and c.get("sm_max_mhz") and c["sm_mhz"] < 0.8 * c["sm_max_mhz"] and not c.get("reasons"):
        return False
    return True


def timed_loop(step, steps, stream, local, barrier):
    """K timed steps bracketed by barrier + synchronize, CUDA events on the launching stream, nvidia-smi clocks
    sampled during the region; re-measured once if the clock record breaks the timing rules."""
    import torch
    import paper_2204_05586_b200 as ss
    for attempt in range(2):
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        launches0 = ss.kernel_launches()
        with ClockSampler(local) as clk:
            # ≈ 1 ms device-side spin before the region: the host enqueues the first steps meanwhile, so no event of
            # the region waits on host launch latency (matters only for sub-millisecond steps such as C2's)
            torch.cuda._sleep(2_000_000)
            start.record(stream)
            for i in range(steps):
                step(evs[i])
            end.record(stream)
            torch.cuda.synchronize()
        launches = ss.kernel_launches() - launches0
        barrier()
        clocks = clk.summary()
        if attempt:
            clocks["remeasured"] = True
        bad = 0.0 if clocks_ok(clocks) else 1.0
        if torch.distributed.is_available() and torch.distributed.is_initialized():
            # collective decision: every rank re-measures or none
            bad = reduce_max([bad], "cuda", torch.distributed.get_world_size())[0]
        if not bad:
            break
    return start.elapsed_time(end), evs, launches, clocks


def dist_setup(n_gpus: int):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != n_gpus and world > 1:
        raise SystemExit(f"--gpus {n_gpus} but WORLD_SIZE={world}")
    return rank, world, local


def cpu_model() -> str:
    """Host CPU model (state the core count and CPU model beside the CPU baseline)."""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_oracle_sample(w: W.Workload, target_s: float):
    """Time the oracle (double instantiation, all host cores) on a bounded sample of workload w: sweeps strided
    across the batch, each over its first k_end intervals, sized from a calibration run to ≈ target_s seconds."""
    import oracle
    oracle.build()
    cores = os.cpu_count() or 1

    def run(n_sweeps, k_end):
        idx = np.linspace(0, w.batch - 1, n_sweeps).astype(int)
        t = time.perf_counter()
        oracle.evaluate(w.spin, w.method, w.expo, w.tau, w.frame, w.field, sweep=w.sweep[idx], t0=w.t0, t1=w.t1,
                        dt_int=w.dt_int, dt_out=w.dt_out, psi0=w.psi0[idx], long_double=False,
                        want_unitaries=False, nthreads=cores, k_begin=0, k_end=k_end)
        return time.perf_counter() - t, n_sweeps * k_end * w.L

    n_sw = min(w.batch, max(1, cores))
    k_cal = max(1, min(w.K, 64))
    dt_cal, steps_cal = run(n_sw, k_cal)
    rate = steps_cal / max(dt_cal, 1e-6)
    want_steps = rate * target_s
    k_end = int(min(w.K, max(1, want_steps / (n_sw * w.L))))
    if k_end == w.K and n_sw < w.batch:
        n_sw = int(min(w.batch, max(n_sw, want_steps / (w.K * w.L))))
    return run, n_sw, k_end, cores


def run_reference(args, rank, world):
    """The reference arm of this tier: the CPU oracle, timed as it stands on the host cores (rank 0 only)."""
    if rank != 0:
        return
    w = get_workload(args.workload, args.batch, args.expo)
    run, n_sw, k_end, cores = cpu_oracle_sample(w, target_s=args.ref_step_seconds)
    for _ in range(args.warmup):
        run(n_sw, k_end)
    times, steps = [], 0
    for _ in range(args.steps):
        dt, n = run(n_sw, k_end)
        times.append(dt)
        steps += n
    total = sum(times)
    value = steps / total
    sample = (f"{n_sw} of {w.batch} sweeps (evenly strided) x first {k_end} of {w.K} intervals x L={w.L} "
              f"= {n_sw * k_end * w.L} fine steps per step; oracle<double>, std::thread x {cores}")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config_of(w, args, world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample,
                             "cpu": cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_of(w: W.Workload, args, world):
    return {"workload": w.name, "spin": w.spin, "exponentiator": w.expo, "trotter_cutoff": w.tau,
            "integration": w.method, "rotating_frame": w.frame, "field": w.field, "time_end": w.t1,
            "time_step_integration": w.dt_int, "time_step_output": w.dt_out, "K": w.K, "L": w.L,
            "batch_per_rank": w.batch, "global_batch": w.batch * world if args.scaling == "weak" else args.batch,
            "parallelism": f"sweep-shard x{world}", "l2": "no flush: per-step working set (U + states) >> 126 MB L2"}


def reduce_max(vals, dev, world):
    """MAX over ranks (NCCL: on the device; gloo: on the host)."""
    import torch
    if world == 1:
        return list(vals)
    t = torch.tensor(vals, dtype=torch.float64,
                     device=dev if torch.distributed.get_backend() == "nccl" else "cpu")
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return t.tolist()


def shard_of(args, rank, world):
    """This rank's contiguous block [lo, hi) of sweeps and the whole job's workload (shards are
    contiguous blocks of B/G sweeps).  With --emulate-ranks N on one process: rank 0's block of an N-rank job."""
    ranks = world
    if world == 1 and args.emulate_ranks > 1:
        ranks = args.emulate_ranks
    if args.scaling == "weak":
        full = get_workload(args.workload, args.batch * ranks, args.expo)
        return rank * args.batch, (rank + 1) * args.batch, full
    full = get_workload(args.workload, args.batch, args.expo)
    per = (full.batch + ranks - 1) // ranks
    return rank * per, min(full.batch, (rank + 1) * per), full


def paper_benchmark(args, dev, steps: int = 20):
    """The paper's own benchmark (C2: one spin-one Eq. neural_pulse simulation, 100 ms at δt = 100 ns, P:866-870;
    SURVEY §8(d) reports it beside C3) timed after the headline line's timed region, so the default run shows it:
    device fine steps/s and the interval kernel's counted-flop fraction of the FP64 peak."""
    import torch
    import paper_2204_05586_b200 as ss
    w = get_workload("C2", 1)
    sim = ss.Simulator(w.spin, w.method, w.expo, w.tau, w.frame, args.precision, w.field)
    sweep, psi0 = torch.from_numpy(w.sweep).to(dev), torch.from_numpy(w.psi0).to(dev)
    states = torch.empty((1, w.K + 1, w.dim), dtype=torch.complex128, device=dev)
    ws = torch.empty(sim.workspace_bytes(1, w.K, True), dtype=torch.uint8, device=dev)
    sim.evaluate(sweep, w.t0, w.t0 + w.dt_out, w.dt_int, w.dt_out, psi0, want_unitaries=False)
    sim.set_validation(False)
    stream = torch.cuda.current_stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    t_int = []
    for i in range(3 + steps):
        if i == 3:
            torch.cuda.synchronize()
            ev[0].record(stream)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record(stream)
        sim.set_split_event(e[1])
        sim.evaluate(sweep, w.t0, w.t1, w.dt_int, w.dt_out, psi0, want_unitaries=False, workspace=ws, out_states=states)
        sim.set_split_event(None)
        e[2].record(stream)
        if i >= 3:
            t_int.append(e)
    ev[1].record(stream)
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / steps
    ms_int = float(np.mean([e[0].elapsed_time(e[1]) for e in t_int]))
    flops = algorithmic_flops_per_fine_step(w.spin, w.expo, w.tau, w.method) * w.fine_steps
    return {"workload": "C2", "value": w.fine_steps / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms, "steps": steps,
            "interval_ms": ms_int, "roofline_frac": flops / (ms_int * 1e-3) / 1e12 / FP64_PEAK_TFLOPS,
            "note": "one simulation of 1e5 intervals x 10 steps (2.6 waves of interval threads); timed after the "
                    "headline's timed region"}


def run_ours(args, rank, world, local):
    import torch
    import paper_2204_05586_b200 as ss

    gpu = 0 if args.share_gpu else local
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    if world > 1:
        import torch.distributed as dist
        if args.dist_backend == "nccl":
            os.environ.setdefault("NCCL_DEBUG", "INFO")   # the init log names the communicator (comm_nranks)
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    if args.workload == "C4":
        return run_time_partition(args, rank, world, local, dev)
    # sweep shard of this rank
    lo, hi, full = shard_of(args, rank, world)
    w = full.with_(sweep=np.ascontiguousarray(full.sweep[lo:hi]), psi0=np.ascontiguousarray(full.psi0[lo:hi]))
    B, K, L, D = w.batch, w.K, w.L, w.dim
    sim = ss.Simulator(w.spin, w.method, w.expo, w.tau, w.frame, args.precision, w.field)
    sweep = torch.from_numpy(w.sweep).to(dev)
    psi0 = torch.from_numpy(w.psi0).to(dev)
    states = torch.empty((B, K + 1, D), dtype=torch.complex128, device=dev)
    ws = torch.empty(sim.workspace_bytes(B, K, True), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    # The step is the public ss_evaluate call (interval kernel + state scan; U_k not requested, so it stays in the
    # workspace — compact SU(2) elements on the SU(2)-form paths).  Its synchronous input validation runs once here,
    # on the full inputs, and is then switched off (ss_set_validation: a one-time check, not part of the path).
    sim.evaluate(sweep, w.t0, w.t0 + w.dt_out, w.dt_int, w.dt_out, psi0, want_unitaries=False)
    sim.set_validation(False)

    def step(ev=None):
        if ev is not None:
            ev[0].record(stream)
            sim.set_split_event(ev[1])       # recorded inside ss_evaluate between the interval kernel and the scan
        sim.evaluate(sweep, w.t0, w.t1, w.dt_int, w.dt_out, psi0, want_unitaries=False, workspace=ws,
                     out_states=states)
        if ev is not None:
            ev[2].record(stream)
            sim.set_split_event(None)

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    elapsed_ms, evs, launches, clocks = timed_loop(step, args.steps, stream, local, barrier)
    t_interval = float(np.mean([e[0].elapsed_time(e[1]) for e in evs]))
    t_scan = float(np.mean([e[1].elapsed_time(e[2]) for e in evs]))
    per_step = [e[0].elapsed_time(e[2]) for e in evs]          # best and median step beside the mean
    best, med = float(np.min(per_step)), float(np.median(per_step))
    elapsed_ms, t_interval, t_scan, best, med = reduce_max([elapsed_ms, t_interval, t_scan, best, med], dev, world)
    steps_per_rank = w.fine_steps
    emulated = world == 1 and args.emulate_ranks > 1
    total_steps = steps_per_rank * world if (args.scaling == "weak" or emulated) else full.fine_steps
    value = total_steps * args.steps / (elapsed_ms * 1e-3)

    # roofline of the dominant kernel (interval kernel): algorithmic flops per launch / average launch duration
    flops_launch = algorithmic_flops_per_fine_step(w.spin, w.expo, w.tau, w.method) * steps_per_rank
    achieved = flops_launch / (t_interval * 1e-3) / 1e12
    scan_bpi = scan_bytes_per_interval(D, su2_form(w))
    scan_gbs = B * K * scan_bpi / (t_scan * 1e-3) / 1e9
    peak = FP64_PEAK_TFLOPS if args.precision == "fp64" else FP32_PEAK_TFLOPS
    kernel_name = f"interval_kernel<spin-{w.spin},{w.expo},{w.method},{w.field},{args.precision}>"

    # e2e through the C ABI with HOST buffers (pinned), copies inside the timed region
    e2e = None
    if not args.no_e2e:
        h_sweep = torch.from_numpy(w.sweep).pin_memory().numpy()
        h_psi0 = torch.from_numpy(w.psi0).pin_memory().numpy()
        h_states = torch.empty((B, K + 1, D), dtype=torch.complex128).pin_memory().numpy()
        sim.evaluate_host(h_sweep, w.t0, w.t1, w.dt_int, w.dt_out, h_psi0, out_states=h_states, n_chunks=args.chunks)
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            sim.evaluate_host(h_sweep, w.t0, w.t1, w.dt_int, w.dt_out, h_psi0, out_states=h_states,
                              n_chunks=args.chunks)
        e2e_s = time.perf_counter() - t0
        e2e_s = reduce_max([e2e_s], dev, world)[0]
        e2e = {"value": total_steps * args.steps / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": int(h_sweep.nbytes + h_psi0.nbytes), "d2h_bytes_per_step": int(h_states.nbytes),
               "n_chunks": args.chunks}

    measured_peak = None
    if rank == 0 and not args.no_probe:
        try:
            from tools import build_tools
            measured_peak = build_tools.probe()[0]
        except Exception as exc:  # probe is context only
            measured_peak = f"unavailable: {exc}"

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        run, n_sw, k_end, cores = cpu_oracle_sample(w, target_s=args.cpu_seconds)
        dt, n = run(n_sw, k_end)
        cpu = {"value": n / dt, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu": cpu_model(),
               "sample": f"{n_sw} of {B} sweeps x first {k_end} of {K} intervals x L={L} = {n} fine steps, "
                         f"oracle<double>, std::thread x {cores}, {dt:.1f} s"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64" if args.precision == "fp64" else "f32",
            "data": "synthetic", "config": config_of(w, args, world),
            "roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": ncu_traffic(kernel_name, w.name, B == 8192),
                         "kernel": kernel_name,
                         "flops_per_launch": flops_launch, "ms_per_launch": t_interval,
                         "dense_equivalent_tflops": dense_equivalent_flops_per_fine_step(w.spin, w.expo, w.tau, w.method)
                         * steps_per_rank / (t_interval * 1e-3) / 1e12,
                         "peak_basis": ("nominal FP64: 148 SM x 64 DFMA/clk x 2 x 1.965 GHz (DESIGN.md §6)"
                                        if args.precision == "fp64" else
                                        "nominal FP32: 148 SM x 128 FFMA/clk x 2 x 1.965 GHz (DESIGN.md §6)"),
                         "measured_dfma_peak_tflops": measured_peak,
                         # the same achieved rate against the DFMA microbenchmark's sustainable peak, and the rate of
                         # the flops the kernel actually executes (ncu SASS counts) against the nominal peak
                         "frac_of_measured_dfma_peak": (achieved / measured_peak
                                                        if isinstance(measured_peak, float) and measured_peak > 0
                                                        else None),
                         "executed": executed_of(kernel_name, w.name, steps_per_rank, t_interval, peak),
                         "frac_at_observed_clock": (achieved / (peak * clocks["sm_mhz"] / SM_MAX_MHZ)
                                                    if clocks.get("sm_mhz") else None)},
            "scan": {"bound": "hbm", "achieved": scan_gbs, "unit": "GB/s", "peak": hbm_peak_gbs()[0],
                     "frac": scan_gbs / hbm_peak_gbs()[0], "peak_basis": hbm_peak_gbs()[1], "ms_per_launch": t_scan,
                     "bytes_per_launch": B * K * scan_bpi,
                     "operators": "SU(2) elements, 32 B" if su2_form(w) else f"dense {D}x{D} complex128"},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches), "clocks": clocks,
            "fine_steps_per_step": total_steps,
            "step_ms": {"mean": elapsed_ms / args.steps, "best": best, "median": med,
                        "note": "best/median of the per-step events (interval kernel start to state pass end); "
                                "mean = the bracketed region / K"},
        }
        if world == 1 and args.workload == "C3" and not emulated and not args.no_secondary:
            line["paper_benchmark"] = paper_benchmark(args, dev)
        if emulated:
            line["emulated"] = {"ranks": args.emulate_ranks, "rank": 0, "sweeps_per_rank": B,
                                "predicted_value": value * args.emulate_ranks,
                                "note": "one GPU timing rank 0's shard; value is that shard's rate, predicted_value "
                                        "assumes the other ranks' identical shards run concurrently (no exchange)"}
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def run_time_partition(args, rank, world, local, dev):
    """C4: one long spin-half simulation (1 s at δt = 1 ns, K = 1e6) time-partitioned over the ranks: each rank
    computes its intervals (global k), reduces them to its aggregate, the aggregates are all-gathered over NCCL
    (the only exchange, 64 B per rank), each rank composes its carry and scans its own intervals (strong scaling)."""
    import torch
    import paper_2204_05586_b200 as ss
    from paper_2204_05586_b200.distributed import gather_aggregates, partition_bounds

    w = get_workload("C4", 1)
    K, L, D = w.K, w.L, w.dim
    # --emulate-ranks N on one GPU: rank 0's slice of an N-rank partition (its aggregate is computed, the exchange is
    # not: a µs-scale all-gather of 64 B per rank)
    ranks = args.emulate_ranks if world == 1 and args.emulate_ranks > 1 else world
    kb, kc = partition_bounds(K, ranks, rank)
    sim = ss.Simulator(w.spin, w.method, w.expo, w.tau, w.frame, args.precision, w.field)
    sweep = torch.from_numpy(w.sweep).to(dev)
    psi0 = torch.from_numpy(w.psi0).to(dev)
    U = torch.empty((1, kc, D, D), dtype=torch.complex128, device=dev)
    states = torch.empty((1, kc + 1, D), dtype=torch.complex128, device=dev)
    lib = ss._lib.load()
    scan_ws = torch.empty(int(lib.ss_scan_workspace_bytes(D, 1, kc)), dtype=torch.uint8, device=dev)
    A_zero = torch.zeros((1, D, D), dtype=torch.complex128, device=dev)
    stream = torch.cuda.current_stream()
    sim.evaluate(sweep, w.t0, w.t0 + 20 * w.dt_out, w.dt_int, w.dt_out, psi0)     # validation + warm-up

    def step(ev=None):
        if ev is not None:
            ev[0].record(stream)
        sim.compute_unitaries(sweep, w.t0, w.t1, w.dt_int, w.dt_out, k_begin=kb, k_count=kc, out=U)
        if ev is not None:
            ev[1].record(stream)
        # the last partition's aggregate feeds no carry: it contributes zeros to the all-gather
        A = ss.chain_aggregate(U) if rank < ranks - 1 else A_zero
        A_all = gather_aggregates(A) if world > 1 else A[None]
        carry = ss.compose_carry(A_all, psi0, rank)
        ss.scan_states(U, carry, out=states, workspace=scan_ws)
        if ev is not None:
            ev[2].record(stream)

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    elapsed_ms, evs, launches, clocks = timed_loop(step, args.steps, stream, local, barrier)
    t_interval = float(np.mean([e[0].elapsed_time(e[1]) for e in evs]))
    t_rest = float(np.mean([e[1].elapsed_time(e[2]) for e in evs]))
    elapsed_ms, t_interval, t_rest = reduce_max([elapsed_ms, t_interval, t_rest], dev, world)
    # e2e at N = 1: the single simulation through the host-buffer C-ABI call (pinned; H2D of the sweep and ψ0, D2H of
    # all 1e6 + 1 states inside the timed region), pipelined over --c4-chunks time chunks.  A time partition over N > 1 ranks has no host-buffer entry point.
    e2e = None
    if world == 1 and not args.no_e2e:
        h_sweep = torch.from_numpy(w.sweep).pin_memory().numpy()
        h_psi0 = torch.from_numpy(w.psi0).pin_memory().numpy()
        h_states = torch.empty((1, K + 1, D), dtype=torch.complex128).pin_memory().numpy()
        sim.evaluate_host(h_sweep, w.t0, w.t1, w.dt_int, w.dt_out, h_psi0, out_states=h_states, n_chunks=args.c4_chunks)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            sim.evaluate_host(h_sweep, w.t0, w.t1, w.dt_int, w.dt_out, h_psi0, out_states=h_states, n_chunks=args.c4_chunks)
        e2e_s = time.perf_counter() - t0
        e2e = {"value": w.fine_steps * args.steps / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": int(h_sweep.nbytes + h_psi0.nbytes), "d2h_bytes_per_step": int(h_states.nbytes),
               "n_chunks": args.c4_chunks}
    value = w.fine_steps * args.steps / (elapsed_ms * 1e-3)
    flops_launch = algorithmic_flops_per_fine_step(w.spin, w.expo, w.tau, w.method) * kc * L
    achieved = flops_launch / (t_interval * 1e-3) / 1e12
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64" if args.precision == "fp64" else "f32",
            "data": "synthetic",
            "config": {"workload": "C4", "spin": "half", "field": w.field, "time_end": w.t1,
                       "time_step_integration": w.dt_int, "time_step_output": w.dt_out, "K": K, "L": L,
                       "parallelism": f"time-partition x{world} (NCCL all_gather of carry aggregates)",
                       "k_per_rank": kc},
            "roofline": {"bound": "alu", "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                         "frac": achieved / FP64_PEAK_TFLOPS, "traffic": None,
                         "kernel": f"interval_kernel<spin-half,analytic,cf4,neural,{args.precision}>",
                         "flops_per_launch": flops_launch, "ms_per_launch": t_interval,
                         "peak_basis": "nominal FP64: 148 SM x 64 DFMA/clk x 2 x 1.965 GHz (DESIGN.md §6)",
                         "executed": executed_of(f"interval_kernel<spin-half,analytic,cf4,neural,{args.precision}>",
                                                 "C4", kc * L, t_interval, FP64_PEAK_TFLOPS)},
            "interval_ms_per_launch": t_interval, "exchange_and_scan_ms": t_rest, "e2e": e2e,
            "gpu_launches": int(launches), "clocks": clocks,
        }
        if ranks != world:
            line["value"] = kc * L * args.steps / (elapsed_ms * 1e-3)
            line["emulated"] = {"ranks": ranks, "rank": 0, "k_per_rank": kc,
                                "predicted_value": line["value"] * ranks,
                                "note": "one GPU timing rank 0's time slice (interval kernel, aggregate, carry, scan); "
                                        "value is that slice's rate, predicted_value assumes the other ranks' slices "
                                        "run concurrently and the 64-B all-gather is free"}
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["C3", "C2", "C5", "C4", "G1"], default="C3")
    ap.add_argument("--batch", type=int, default=8192, help="sweeps per rank (weak) or in total (strong), C3")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="strong")
    ap.add_argument("--emulate-ranks", type=int, default=1,
                    help="one GPU: time rank 0's shard of an N-rank strong-scaling job (per-rank shard shapes)")
    ap.add_argument("--precision", choices=["fp64", "fp32"], default="fp64")
    ap.add_argument("--expo", choices=["analytic", "lie_trotter"], default=None,
                    help="C5 only: the exponentiator column of the accuracy/throughput matrix (default lie_trotter)")
    ap.add_argument("--chunks", type=int, default=40,
                    help="chunks of the pipelined host-buffer (e2e) call (time chunks for large batches; 0: automatic)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-step-seconds", type=float, default=8.0)
    ap.add_argument("--c4-chunks", type=int, default=6, help="time chunks of C4's host-buffer (e2e) call")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-probe", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the paper-benchmark (C2) side measurement")
    ap.add_argument("--dist-backend", choices=["nccl", "gloo"], default="nccl",
                    help="gloo only to exercise the multi-rank code path where NCCL cannot run (e.g. ranks sharing a GPU)")
    ap.add_argument("--share-gpu", action="store_true", help="map every rank to cuda:0 (code-path test, not timing)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("note: --warmup < 3 violates the timing rules; using 3", file=sys.stderr)
        args.warmup = 3
    rank, world, local = dist_setup(args.gpus)
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
