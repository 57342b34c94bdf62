#!/usr/bin/env python3
"""DRAM traffic per quote of one batch call, from ncu launch lists.

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \\
        --clock-control none -k regex:<kernels> --csv --log-file traffic_<w>.csv \\
        python bench.py --workload <w> --steps 1 --warmup 0 --no-e2e --no-cpu --no-kernel-timing
    python tools/traffic.py gpurun_out/traffic_c4.csv:c4:100000000 ... [--out profiles/roofline_traffic.json]

Sums dram__bytes_read.sum + dram__bytes_write.sum over every profiled launch
(one call's kernels) and divides by the call's rows; bench.py scales it back
by the rows of a launch for roofline.traffic.
"""
import argparse
import csv
import json
import os
import sys

UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def parse(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = None
    out = []
    for r in rows:
        if "Metric Name" in r:
            hdr = {h: i for i, h in enumerate(r)}
            continue
        if hdr is None or len(r) < len(hdr):
            continue
        out.append((r[hdr["ID"]], r[hdr["Kernel Name"]], r[hdr["Metric Name"]], r[hdr["Metric Unit"]],
                    float(r[hdr["Metric Value"]].replace(",", ""))))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("specs", nargs="+", help="csv:workload:rows")
    ap.add_argument("--out", default=os.path.join(os.path.dirname(__file__), "..", "profiles",
                                                  "roofline_traffic.json"))
    a = ap.parse_args()
    res = json.load(open(a.out)) if os.path.exists(a.out) else {}
    for spec in a.specs:
        path, wl, rows = spec.rsplit(":", 2)
        rows = int(rows)
        by_kernel = {}
        total = 0.0
        for _id, name, metric, unit, val in parse(path):
            if metric.startswith("dram__bytes"):
                b = val * UNIT.get(unit, 1.0)
                total += b
                k = name.split("(")[0]
                by_kernel[k] = by_kernel.get(k, 0.0) + b
        res[wl] = {"dram_bytes_per_quote": total / rows,
                   "per_kernel_bytes_per_quote": {k: v / rows for k, v in sorted(by_kernel.items())},
                   "rows": rows, "source": os.path.basename(path)}
        print(wl, "%.1f B/quote" % (total / rows), file=sys.stderr)
    res["note"] = ("ncu dram__bytes_read.sum + dram__bytes_write.sum over the kernels of one batch "
                   "call, per quote (tools/traffic.py); bench.py reports it x rows as roofline.traffic")
    json.dump(res, open(a.out, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
