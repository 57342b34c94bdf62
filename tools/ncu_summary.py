#!/usr/bin/env python3
"""Summarise an `ncu --set full` report: per kernel launch, duration, occupancy,
issue and FP64-pipe utilisation, DRAM bytes and the top stall reasons.

    python tools/ncu_summary.py gpurun_out/prof_X.ncu-rep > profiles/rN_ncu_X.txt
"""
import csv
import io
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum",
    "launch__grid_size",
    "launch__registers_per_thread",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
]
STALLS = ["long_scoreboard", "wait", "selected", "short_scoreboard", "not_selected", "branch_resolving",
          "no_instruction", "math_pipe_throttle", "lg_throttle", "mio_throttle", "barrier", "dispatch_stall"]


def main():
    rep = sys.argv[1]
    mets = METRICS + ["smsp__average_warps_issue_stalled_%s_per_issue_active.ratio" % s for s in STALLS]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(mets)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    units = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    for r in rows[2:]:
        print("== %s" % r[ix["Kernel Name"]])
        for m in METRICS:
            if m in ix:
                print("  %s = %s %s" % (m, r[ix[m]], units[ix[m]]))
        st = []
        for s in STALLS:
            k = "smsp__average_warps_issue_stalled_%s_per_issue_active.ratio" % s
            if k in ix and r[ix[k]]:
                st.append((float(r[ix[k]].replace(",", "")), s))
        st.sort(reverse=True)
        print("  stall cycles per issued instruction: " + ", ".join("%s=%.2f" % (s, v) for v, s in st[:8]))


if __name__ == "__main__":
    main()
