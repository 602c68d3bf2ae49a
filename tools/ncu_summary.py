"""Summarise an ncu report (--set full) into the handful of numbers the roofline story needs, as text for profiles/.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/r01/ncu_<kernel>.txt
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("kernel", "Kernel Name"),
    ("duration_ms", "gpu__time_duration.sum"),
    ("sm_clock_ghz", "sm__cycles_elapsed.avg.per_second"),
    ("registers_per_thread", "launch__registers_per_thread"),
    ("grid", "launch__grid_size"),
    ("block", "launch__block_size"),
    ("warps_active_per_sm", "sm__warps_active.avg.per_cycle_active"),
    ("fp64_pipe_active_pct", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
    ("fma_pipe_active_pct", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
    ("issue_active_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
    ("dram_read_bytes", "dram__bytes_read.sum"),
    ("dram_write_bytes", "dram__bytes_write.sum"),
    ("dram_throughput_pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("dfma_thread_inst", "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"),
    ("dmul_thread_inst", "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum"),
    ("dadd_thread_inst", "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"),
    ("ffma_thread_inst", "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum"),
    ("warp_inst_executed", "smsp__inst_executed.sum"),
]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    for vals in rows[2:]:
        d = dict(zip(head, vals))
        u = dict(zip(head, units))
        print(f"# {path}")
        for name, key in KEYS:
            if key in d:
                print(f"{name:24s} {d[key]} {u.get(key, '')}".rstrip())
        stalls = {k[len("smsp__pcsamp_warps_issue_stalled_"):]: float(v) for k, v in d.items()
                  if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")
                  and v not in ("", "0")}
        tot = sum(stalls.values()) or 1.0
        print("stall samples (share):  " + ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in
                                                   sorted(stalls.items(), key=lambda x: -x[1])[:8]))
        print()


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
