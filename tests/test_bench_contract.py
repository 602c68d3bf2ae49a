"""bench.py's JSON-line contract: every key the driver reads is present and well-formed.  The reference arm runs on
CPU; the device arm needs the GPU."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config"}


def run(args, timeout=900):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_contract():
    d = run(["--impl", "reference", "--steps", "1", "--warmup", "0", "--ref-step-seconds", "1"])
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["higher_is_better"] is True and d["value"] > 0
    assert d["metric"] == json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
    assert d["config"]["workload"] == "C3" and "model" not in d["config"]
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_device_arm_contract():
    d = run(["--steps", "2", "--warmup", "3", "--batch", "512", "--cpu-seconds", "2"])
    assert BASE_KEYS <= set(d)
    assert d["dtype"] == "f64" and d["data"] == "synthetic" and d["n_gpus"] == 1 and d["scaling"] in ("weak", "strong")
    rf = d["roofline"]
    assert rf["bound"] == "alu" and rf["unit"] == "TFLOP/s" and 0 < rf["frac"] < 1.0
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-12
    assert d["scan"]["bound"] == "hbm" and d["scan"]["achieved"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    # interval kernel + state scan per step (+ the coarse scan when the fused path runs: 512 × 1e4 intervals is ≥ 16
    # waves at 4 intervals per thread, DESIGN.md §5 item 16)
    assert d["gpu_launches"] in (2 * d["steps"], 3 * d["steps"])
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    pb = d["paper_benchmark"]                      # the paper's own benchmark (C2) beside the headline
    assert pb["workload"] == "C2" and pb["value"] > 0 and 0 < pb["roofline_frac"] < 1.0


def test_flop_model():
    """The per-fine-step flop counts bench.py reports, re-derived from the instruction mix of each
    formulation: scaled double-angle symmetric squaring 24 DFMA + 12 DMUL + 3 DADD = 63 flop (also on the
    tridiagonalised su(3) factor, plus its conjugation by W: 24 complex multiply-adds × 8 = 192), 3×3 residual product
    219, SU(2) group-law product 16 DFMA + 4 DADD = 36."""
    sys.path.insert(0, ROOT)
    import bench
    sym, conj3, prod3, prod2 = 2 * 24 + 12 + 3, 24 * 8, 219, 2 * 16 + 4
    assert bench.algorithmic_flops_per_fine_step("one", "lie_trotter", 24) == 2 * (24 * sym + prod3)
    assert bench.algorithmic_flops_per_fine_step("one", "lie_trotter_su3", 24) == 2 * (24 * sym + conj3 + prod3)
    half = 163                         # ncu-executed per spin-half C4 step (2 × (9 + prod2) = 90 of it in the products)
    assert 2 * (9 + prod2) < half
    assert bench.algorithmic_flops_per_fine_step("half", "analytic", 24) == half
    assert bench.algorithmic_flops_per_fine_step("one", "analytic", 24) == half      # SU(2) accumulation + D¹ map
