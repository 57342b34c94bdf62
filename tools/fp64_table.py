#!/usr/bin/env python3
"""FP64 instruction accounting per workload call from tools/gpu_fp64.sh's ncu
CSVs: thread-level DADD + DMUL + DFMA with the predicate on (the lanes that did
the work), per quote, against the reference's weighted op count W (SURVEY
8(d)); and the rate those instructions ran at against the FP64 pipe's peak.

    python tools/fp64_table.py gpurun_out > profiles/r2/fp64_accounting.json
"""
import collections
import csv
import json
import os
import sys

ROWS = {"c4": 10_000_000, "c1": 1_000_000, "c2": 10_000_000, "c3": 10_000_000, "c5": 10_000_000,
        "rt": 10_000_000}
W = {"c4": 1443.0, "c1": 1405.0, "c2": 1476.0, "c3": 298.0, "c5": 347.0, "rt": 1676.0}
UNIT = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}
PEAK = 17.07e12          # measured DFMA issue rate (fv_probe_fp64_peak): FP64 lane-ops/s


def main(d):
    out = {}
    for w in ROWS:
        p = os.path.join(d, f"fp64_{w}.csv")
        if not os.path.exists(p):
            continue
        rows = [r for r in csv.reader(open(p)) if r]
        hdr = None
        per = collections.defaultdict(dict)
        for r in rows:
            if "Kernel Name" in r:
                hdr = {h: i for i, h in enumerate(r)}
                continue
            if not hdr or len(r) < len(hdr):
                continue
            key = (r[hdr["ID"]], r[hdr["Kernel Name"]].split("(")[0])
            v = float(r[hdr["Metric Value"]].replace(",", ""))
            if r[hdr["Metric Name"]] == "gpu__time_duration.sum":
                v *= UNIT[r[hdr["Metric Unit"]]]
            per[key][r[hdr["Metric Name"]]] = v
        tot = collections.Counter()
        kern = collections.defaultdict(collections.Counter)
        for (i, k), m in per.items():
            f64 = sum(m.get(f"smsp__sass_thread_inst_executed_op_{o}_pred_on.sum", 0) for o in ("dadd", "dmul", "dfma"))
            for name, v in (("fp64_thread_inst", f64), ("time_s", m.get("gpu__time_duration.sum", 0)),
                            ("fp64_warp_inst", m.get("smsp__inst_executed_pipe_fp64.sum", 0)),
                            ("warp_inst", m.get("smsp__inst_executed.sum", 0)),
                            ("thread_inst", m.get("smsp__thread_inst_executed.sum", 0))):
                tot[name] += v
                kern[k][name] += v
        n = ROWS[w]
        out[w] = {
            "rows": n, "W_weighted_ops_per_quote": W[w],
            "fp64_thread_inst_per_quote": tot["fp64_thread_inst"] / n,
            "fp64_inst_over_W": tot["fp64_thread_inst"] / n / W[w],
            "fp64_share_of_thread_inst": tot["fp64_thread_inst"] / max(tot["thread_inst"], 1),
            "lanes_per_fp64_warp_inst": tot["fp64_thread_inst"] / max(tot["fp64_warp_inst"], 1),
            "serialised_kernel_time_ms": tot["time_s"] * 1e3,
            "fp64_rate_T_per_s": tot["fp64_thread_inst"] / tot["time_s"] / 1e12,
            "fp64_rate_frac_of_peak": tot["fp64_thread_inst"] / tot["time_s"] / PEAK,
            "kernels": {k: {"time_ms": v["time_s"] * 1e3, "fp64_thread_inst_per_quote": v["fp64_thread_inst"] / n,
                            "fp64_frac_of_peak": (v["fp64_thread_inst"] / v["time_s"] / PEAK) if v["time_s"] else None}
                        for k, v in sorted(kern.items(), key=lambda kv: -kv[1]["time_s"])},
        }
    out["note"] = ("ncu, one call per workload, kernels serialised (cold caches, side-stream branches in "
                   "sequence); fp64 thread instructions = DADD + DMUL + DFMA with the predicate on; "
                   "peak = the measured DFMA issue rate 17.07 T lane-ops/s; C4 on a 10M-row strided sample")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out")
