"""C-ABI checks that need no GPU: the library builds for sm_100a, loads, exports every symbol include/*.h declares,
rejects bad arguments synchronously, and fails loudly (no CPU fallback) when no CUDA device is present."""
import ctypes
import glob
import os
import re
import subprocess

import numpy as np
import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2204_05586_b200 import build, _lib
    build.build()
    return _lib.load()


def header_symbols():
    syms = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(h).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for m in re.finditer(r"^\s*[A-Za-z_][\w\s\*]*?\b(ss_\w+)\s*\(", text, flags=re.M):
            syms.add(m.group(1))
    return syms


def test_header_declares_the_binding_exports():
    from paper_2204_05586_b200 import _lib
    assert header_symbols() == set(_lib.EXPORTS)


def test_library_exports_every_header_symbol(lib):
    so = os.path.join(ROOT, "paper_2204_05586_b200", "libspinsim_b200.so")
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True, check=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if l.strip()}
    missing = header_symbols() - exported
    assert not missing, missing
    for s in header_symbols():
        assert hasattr(lib, s)


def test_library_is_sm100a_only(lib):
    so = os.path.join(ROOT, "paper_2204_05586_b200", "libspinsim_b200.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_\d+a?", out))
    assert archs == {"sm_100a"}, archs
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    assert "DFMA" in sass                     # FP64 FMA pipe carries the stepper
    assert "HMMA" not in sass                 # no legacy tensor-core path


def test_version_and_params(lib):
    assert lib.ss_version() == 102
    from paper_2204_05586_b200 import num_sweep_params
    assert [num_sweep_params(f) for f in ("constant", "rabi_linear", "rabi_circular", "neural", "gradient",
                                          "su3_constant", "su3_drive")] == [4, 2, 2, 7, 2, 8, 6]
    assert lib.ss_num_sweep_params(99) < 0


def test_plan(lib):
    from paper_2204_05586_b200 import plan, SpinsimError
    assert plan(0.0, 0.1, 100e-9, 1e-6) == (100000, 10, 1e-7)
    assert plan(0.0, 1.0, 1e-9, 1e-6)[:2] == (1000000, 1000)
    with pytest.raises(SpinsimError, match="not an integer"):
        plan(0.0, 0.1, 300e-9, 1e-6)
    with pytest.raises(SpinsimError, match="exceed"):
        plan(1.0, 0.5, 1e-7, 1e-6)
    with pytest.raises(SpinsimError):
        plan(0.0, float("nan"), 1e-7, 1e-6)


def test_create_validation(lib):
    from paper_2204_05586_b200 import Simulator, SpinsimError
    from paper_2204_05586_b200._lib import SS_ERR_UNSUPPORTED, SS_ERR_INVALID
    with pytest.raises(SpinsimError) as e:
        Simulator(spin="half", exponentiation="lie_trotter")
    assert e.value.code == SS_ERR_UNSUPPORTED
    with pytest.raises(SpinsimError) as e:
        Simulator(spin="one", trotter_cutoff=61)
    assert e.value.code == SS_ERR_INVALID
    for spin, expo in (("half", "analytic"), ("one", "lie_trotter"), ("one", "analytic")):
        for method in ("cf4", "midpoint", "heun"):
            for field in ("constant", "rabi_linear", "rabi_circular", "neural", "gradient"):
                for prec in ("fp64", "fp32"):
                    Simulator(spin, method, expo, 24, True, prec, field)      # every instance exists
    # general spin-one exponentiator: every field, and the su(3) fields only with it (readings R19, R20)
    for method in ("cf4", "midpoint", "heun"):
        for field in ("constant", "rabi_linear", "rabi_circular", "neural", "gradient", "su3_constant", "su3_drive"):
            for prec in ("fp64", "fp32"):
                assert Simulator("one", method, "lie_trotter_su3", 24, True, prec, field).num_coefficients == 8
    for expo in ("lie_trotter", "analytic"):
        with pytest.raises(SpinsimError) as e:
            Simulator("one", "cf4", expo, 24, True, "fp64", "su3_drive")
        assert e.value.code == SS_ERR_UNSUPPORTED
    with pytest.raises(SpinsimError) as e:
        Simulator("half", "cf4", "lie_trotter_su3", 24, True, "fp64", "constant")
    assert e.value.code == SS_ERR_UNSUPPORTED
    assert Simulator("one").num_coefficients == 4
    # FP32 needs the rotating frame: in the lab frame its rounding accumulates past the 1e-4 bar
    for spin, expo in (("half", "analytic"), ("one", "lie_trotter"), ("one", "analytic"), ("one", "lie_trotter_su3")):
        for method in ("cf4", "midpoint", "heun"):
            with pytest.raises(SpinsimError) as e:
                Simulator(spin, method, expo, 24, False, "fp32", "constant")
            assert e.value.code == SS_ERR_UNSUPPORTED and "use_rotating_frame" in str(e.value)
            Simulator(spin, method, expo, 24, False, "fp64", "constant")


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback(lib):
    """Without a CUDA device every compute entry point fails with SS_ERR_CUDA — nothing runs on the CPU."""
    from paper_2204_05586_b200 import Simulator, SpinsimError
    from paper_2204_05586_b200._lib import SS_ERR_CUDA
    sim = Simulator("half", field="rabi_circular")
    sweep = np.array([[1.0, 2.0]])
    with pytest.raises(SpinsimError) as e:
        sim.evaluate_host(sweep, 0.0, 1e-5, 1e-7, 1e-6, np.array([[1, 0]], complex))
    assert e.value.code == SS_ERR_CUDA
    fake = ctypes.c_void_p(256)
    rc = lib.ss_compute_unitaries(sim._h, 0.0, 1e-5, 1e-7, 1e-6, 0, 10, 1, fake, fake, None)
    assert rc == SS_ERR_CUDA
    with pytest.raises(TypeError):
        sim.evaluate(torch.zeros((1, 2), dtype=torch.float64), 0.0, 1e-5, 1e-7, 1e-6,
                     torch.zeros((1, 2), dtype=torch.complex128))


def test_argument_errors_are_synchronous(lib):
    from paper_2204_05586_b200 import Simulator
    from paper_2204_05586_b200._lib import SS_ERR_INVALID
    sim = Simulator("one")
    fake = ctypes.c_void_p(4096)
    # bad interval range
    assert lib.ss_compute_unitaries(sim._h, 0.0, 1e-5, 1e-7, 1e-6, 5, 10, 1, fake, fake, None) == SS_ERR_INVALID
    assert b"outside" in lib.ss_last_error()
    # misaligned pointer
    assert lib.ss_compute_unitaries(sim._h, 0.0, 1e-5, 1e-7, 1e-6, 0, 10, 1, ctypes.c_void_p(4097), fake, None) == SS_ERR_INVALID
    # workspace too small
    assert lib.ss_scan_states(3, 2, 100, fake, fake, fake, fake, 16, None) == SS_ERR_INVALID
    assert b"workspace" in lib.ss_last_error()
    assert lib.ss_compose_carry(3, 1, 2, 2, fake, fake, fake, None) == SS_ERR_INVALID
    assert lib.ss_workspace_bytes(sim._h, 8192, 10000, 1) > 8192 * 10000 * 144


def test_user_field_compiles_without_gpu(lib):
    """NVRTC compile of a user field together with the library's interval kernel (NEXT #5) needs no GPU."""
    from paper_2204_05586_b200 import _lib
    src = b"__device__ void user_field(double t_k, double off, const double* p, double f[4]) { f[2] = p[0]; }"
    for spin, expo, prec in ((1, 0, 0), (2, 1, 0), (2, 1, 1)):
        d = _lib.ss_sim_desc(spin, 0, expo, 24, 1, prec, 0)
        assert lib.ss_compile_user_field(ctypes.byref(d), src, 1) == 0, lib.ss_last_error()
    src8 = b"__device__ void user_field(double t_k, double off, const double* p, double f[8]) { f[2] = p[0]; f[5] = p[1]; }"
    for prec in (0, 1):
        d = _lib.ss_sim_desc(2, 0, 2, 24, 1, prec, 0)
        assert lib.ss_compile_user_field(ctypes.byref(d), src8, 2) == 0, lib.ss_last_error()
    d = _lib.ss_sim_desc(1, 0, 0, 24, 1, 0, 0)
    assert lib.ss_compile_user_field(ctypes.byref(d), b"__device__ void user_field( {", 1) == _lib.SS_ERR_INVALID
    assert b"compilation failed" in lib.ss_last_error()


def test_host_chunk_plan(lib):
    """ss_evaluate_host's pipeline plan (pure host logic; 148 SMs assumed without a GPU): sizes always partition the
    batch or the K intervals; C3 takes the 40-chunk tent, C4 six time chunks, C2 the wave-aligned pair whose first
    chunk is exactly two waves of interval threads (148 SMs × 4 blocks × 128 threads per wave, split S = 2), and an
    explicit single chunk is honoured."""
    import workloads as W
    from paper_2204_05586_b200 import Simulator
    cases = {"C3": (W.c3_batched(), 8192), "C4": (W.c4_long(), 1), "C2": (W.c2_neural(), 1),
             "C5": (W.c5_matrix("lie_trotter", batch=100), 100), "small": (W.c3_batched(batch=5, duration=0.2e-3), 5)}
    plans = {}
    for name, (w, batch) in cases.items():
        sim = Simulator(w.spin, w.method, w.expo, w.tau, w.frame, "fp64", w.field)
        K = int(round((w.t1 - w.t0) / w.dt_out))
        for n in (0, 1, 3, 6, 40):
            kind, sizes = sim.host_chunk_plan(w.t0, w.t1, w.dt_int, w.dt_out, batch, n)
            assert all(x >= 1 for x in sizes), (name, n, sizes)
            assert sum(sizes) == (batch if kind == "batch" else K), (name, n, kind, sizes)
            if n == 1:
                assert (kind, sizes) == ("batch", [batch])
        plans[name] = sim.host_chunk_plan(w.t0, w.t1, w.dt_int, w.dt_out, batch, 0)
    assert plans["C3"][0] == "time" and len(plans["C3"][1]) == 40
    assert plans["C4"][0] == "time" and len(plans["C4"][1]) == 6
    assert plans["C2"] == ("wave_pair", [2 * 148 * 4 * 128 // 2, 100000 - 2 * 148 * 4 * 128 // 2])
    assert plans["small"][0] == "batch"


def test_wrappers_reject_bad_shapes_before_the_library(lib):
    """The Python wrappers check shapes, dtypes and layout before any ctypes call (the library reads raw pointers)."""
    from paper_2204_05586_b200 import Simulator
    sim = Simulator("half", "cf4", "analytic", 24, True, "fp64", "rabi_circular")
    sweep = np.zeros((2, 2))
    psi0 = np.zeros((2, 2), np.complex128)
    with pytest.raises(ValueError, match="sweep"):
        sim.evaluate_host(np.zeros((2, 3)), 0.0, 1e-5, 1e-7, 1e-6, psi0)
    with pytest.raises(ValueError, match="state_init"):
        sim.evaluate_host(sweep, 0.0, 1e-5, 1e-7, 1e-6, np.zeros((3, 2), np.complex128))
    with pytest.raises(ValueError, match="out_states"):
        sim.evaluate_host(sweep, 0.0, 1e-5, 1e-7, 1e-6, psi0, out_states=np.zeros((2, 10, 2), np.complex128))
    with pytest.raises(ValueError, match="out_states"):
        sim.evaluate_host(sweep, 0.0, 1e-5, 1e-7, 1e-6, psi0, out_states=np.zeros((2, 11, 2), np.complex64))
    with pytest.raises(ValueError, match="out_states"):
        sim.evaluate_host(sweep, 0.0, 1e-5, 1e-7, 1e-6, psi0,
                          out_states=np.zeros((2, 2, 11), np.complex128).transpose(0, 2, 1))
    with pytest.raises((TypeError, ValueError)):
        sim.evaluate(torch.zeros(2, 2, dtype=torch.float64), 0.0, 1e-5, 1e-7, 1e-6, torch.zeros(2, 2))


def test_workspace_sizes_cover_every_path(lib):
    """Host-only sizing (no GPU): ss_scan_workspace_bytes is non-decreasing in K below the chain kernel's batch size
    (the fused path's coarse scan over K/ipt runs and the two-pass scan's own coarse scan over ⌈K/4⌉ run the workspace
    sized for K), covers the two-pass scan's run products and run states (≥ ⌈K/4⌉ of each per sweep), and
    ss_workspace_bytes adds the fused region (≥ ⌈K/4⌉ run products and run states per sweep) below 4096 sweeps only."""
    from paper_2204_05586_b200 import Simulator
    rng = np.random.default_rng(3)
    for dim in (2, 3):
        for batch in (1, 7, 100, 4095):
            Ks = np.unique(np.concatenate([np.arange(1, 300), rng.integers(1, 3_000_000, 200)]))
            sizes = [int(lib.ss_scan_workspace_bytes(dim, batch, int(K))) for K in Ks]
            assert all(b >= a for a, b in zip(sizes, sizes[1:])), (dim, batch)
            for K, size in zip(Ks[::17], sizes[::17]):
                if K >= 8:
                    runs = -(-int(K) // 4)
                    assert size >= batch * runs * 16 * (2 + dim)
    sim = Simulator("one", "cf4", "analytic", 24, True, "fp64", "neural")
    for batch, K in ((100, 100_000), (1, 100_000_000 // 32)):
        with_f = sim.workspace_bytes(batch, K, True)
        runs = -(-K // 4)
        assert with_f >= batch * K * 16 * 9 + batch * runs * 16 * (9 + 3)      # U, run products (dense), run states
    assert sim.workspace_bytes(8192, 10_000, True) < 8192 * 10_000 * 16 * 9 * 1.02   # no fused region at 8192
