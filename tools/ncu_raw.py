"""Key raw metrics + top stall reasons of the first kernel in an ncu report.

usage: python tools/ncu_raw.py report.ncu-rep [extra_metric_prefix ...]
"""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum"]


def main(rep, extra):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    for k in KEYS + [x for x in h if any(x.startswith(e) for e in extra)]:
        if k in h:
            i = h.index(k)
            print(f"{k:70s} {v[i]} {u[i]}")
    st = []
    for i, k in enumerate(h):
        if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(v[i]), k.replace("smsp__average_warps_issue_stalled_", "").replace(
                    "_per_issue_active.ratio", "")))
            except ValueError:
                pass
    print("stalls/issue:", ", ".join(f"{k}={x:.2f}" for x, k in sorted(st)[::-1][:8]))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
