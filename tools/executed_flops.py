"""Executed FP64 flops per fine step of the interval kernel, from ncu's SASS op counts (2·DFMA + DMUL + DADD per
thread instruction, predicated-on), one capture per workload on a warm launch (tools/profile_run.py).  Writes the
JSON that bench.py reads into roofline.executed (`profiles/executed_flops.json` once reviewed and copied):

    python tools/executed_flops.py gpurun_out/<tag>          # on the GPU box
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = ["gpu__time_duration.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
           "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"]
# (workload tag, bench kernel name, profile_run arguments, fine steps of one launch)
CASES = [
    ("C3", "interval_kernel<spin-one,lie_trotter,cf4,neural,fp64>", ["--workload", "C3", "--batch", "1024"],
     1024 * 10000 * 10),
    ("C2", "interval_kernel<spin-one,lie_trotter,cf4,neural,fp64>", ["--workload", "C2"], 100000 * 10),
    ("C4", "interval_kernel<spin-half,analytic,cf4,neural,fp64>", ["--workload", "C4", "--duration", "0.1"],
     100000 * 1000),
    ("C5", "interval_kernel<spin-one,analytic,cf4,neural,fp64>", ["--workload", "C5", "--expo", "analytic"],
     100 * 100000 * 10),
    ("G1", "interval_kernel<spin-one,lie_trotter_su3,cf4,su3_drive,fp64>", ["--workload", "G1", "--batch", "1024"],
     1024 * 10000 * 10),
]


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/flops"
    os.makedirs(out, exist_ok=True)
    res = {"_about": "FP64 flops one fine step executes in the interval kernel: (2*DFMA + DMUL + DADD) thread "
                     "instructions / fine steps, ncu SASS counts of one warm launch (tools/executed_flops.py)"}
    for tag, kernel, args, steps in CASES:
        log = os.path.join(out, f"flops_{tag}.csv")
        cmd = ["ncu", "--metrics", ",".join(METRICS), "--clock-control", "none", "-k", "regex:interval_kernel",
               "-s", "1", "-c", "1", "--csv", "--log-file", log, sys.executable,
               os.path.join(ROOT, "tools", "profile_run.py"), *args]
        subprocess.run(cmd, check=True, capture_output=True)
        rows = [r for r in csv.reader(l for l in open(log) if l.startswith('"'))]
        hdr = rows[0]
        m = {r[hdr.index("Metric Name")]: float(r[hdr.index("Metric Value")].replace(",", "")) for r in rows[1:]}
        dfma = m["smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"] / steps
        dmul = m["smsp__sass_thread_inst_executed_op_dmul_pred_on.sum"] / steps
        dadd = m["smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"] / steps
        res[f"{kernel}@{tag}"] = {
            "flops_per_fine_step": 2 * dfma + dmul + dadd, "dfma": dfma, "dmul": dmul, "dadd": dadd,
            "fp64_pipe_pct": m["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"],
            "source": f"profiles/r02/{os.path.basename(os.path.normpath(out))}/flops_{tag}.csv"}
        print(tag, json.dumps(res[f"{kernel}@{tag}"]))
    json.dump(res, open(os.path.join(out, "executed_flops.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
