#!/usr/bin/env python3
"""Copy one tools/gpu_full.sh run (TAG) from gpurun_out/ into profiles/:
bench lines, ncu --set full summaries (LBR, Halley), the launch-list summary
(+ raw, gzipped), per-workload DRAM traffic and roofline_traffic.json.

    python tools/save_evidence.py r1h
"""
import collections
import csv
import gzip
import os
import shutil
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(REPO, "gpurun_out")
P = os.path.join(REPO, "profiles")
ROWS = {"c4": 100_000_000, "c1": 1_000_000, "c2": 10_000_000, "c3": 10_000_000, "c5": 10_000_000,
        "rt": 10_000_000}
UNIT = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
        "s": 1e3, "second": 1e3}


def launches(tag):
    rows = [r for r in csv.reader(open(os.path.join(G, f"launches_{tag}.csv"))) if r]
    hdr, tot, cnt = None, collections.defaultdict(float), collections.Counter()
    for r in rows:
        if "Kernel Name" in r:
            hdr = {h: i for i, h in enumerate(r)}
            continue
        if not hdr or len(r) < len(hdr) or r[hdr["Metric Name"]] != "gpu__time_duration.sum":
            continue
        k = r[hdr["Kernel Name"]].split("(")[0]
        tot[k] += float(r[hdr["Metric Value"]].replace(",", "")) * UNIT[r[hdr["Metric Unit"]]]
        cnt[k] += 1
    lbr = sum(v for k, v in tot.items() if "lbr" in k)
    with open(os.path.join(P, f"{tag}_launches_c4_summary.csv"), "w") as f:
        f.write("# ncu --metrics gpu__time_duration.sum --clock-control none, python bench.py --steps 2 "
                "--warmup 1 --no-e2e --no-cpu (C4 100M; warm-up + 2 timed calls + the per-kernel timing "
                "pass): per-kernel sums over all launches (serialised by ncu, cold-cache per launch -- "
                "compare shares, not absolutes)\nkernel,launches,total_ms,share_of_lbr_call\n")
        for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
            f.write(f"{k},{cnt[k]},{v:.3f},{(v / lbr if 'lbr' in k else 0):.4f}\n")
    with open(os.path.join(G, f"launches_{tag}.csv"), "rb") as src, \
            gzip.open(os.path.join(P, f"{tag}_launches_c4.csv.gz"), "wb") as dst:
        shutil.copyfileobj(src, dst)


def main(tag):
    lines = []
    for suf in ("", "_c1", "_c2", "_c3", "_c5", "_rt", "_ref"):
        path = os.path.join(G, f"bench_{tag}{suf}.json")
        if os.path.exists(path):
            lines.append(open(path).read().strip().splitlines()[-1])
    open(os.path.join(P, f"{tag}_bench_lines.jsonl"), "w").write("\n".join(lines) + "\n")
    for rep, name in (("prof", "lbr"), ("profh", "halley"), ("profg", "price_greeks")):
        src = os.path.join(G, f"{rep}_{tag}.ncu-rep")
        if os.path.exists(src):
            out = subprocess.run([sys.executable, os.path.join(REPO, "tools", "ncu_summary.py"), src],
                                 capture_output=True, text=True).stdout
            open(os.path.join(P, f"{tag}_ncu_{name}.txt"), "w").write(out)
    if os.path.exists(os.path.join(G, f"launches_{tag}.csv")):
        launches(tag)
    for name in (f"api_e2e_{tag}.json", f"pytest_gpu_{tag}.txt", f"smoke_{tag}.txt", f"cpu_{tag}.txt",
                 f"gpu_{tag}.txt"):
        src = os.path.join(G, name)
        if os.path.exists(src):
            shutil.copy(src, os.path.join(P, name))
    specs = []
    for w, n in ROWS.items():
        src = os.path.join(G, f"traffic_{tag}_{w}.csv")
        if os.path.exists(src):
            dst = os.path.join(P, f"{tag}_traffic_{w}.csv")
            shutil.copy(src, dst)
            specs.append(f"{dst}:{w}:{n}")
    if specs:
        subprocess.run([sys.executable, os.path.join(REPO, "tools", "traffic.py")] + specs, check=True)


if __name__ == "__main__":
    main(sys.argv[1])
