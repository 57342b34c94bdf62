#!/usr/bin/env python3
"""Join an ncu SASS source page with nvdisasm line info: per-source-line
dynamic warp instructions, stall samples and instruction mix of one kernel.

    nvdisasm -g -c fv_kernels.sm_100a.cubin > all_g.sass
    ncu -i rep.ncu-rep --page source --csv --print-source sass \
        --kernel-name-base mangled -k regex:<name> > k.csv
    python tools/sass_lines.py all_g.sass <mangled-name> k.csv [--top 40]
"""
import argparse
import collections
import csv
import os
import re


def parse_lineinfo(path, func):
    """address -> (file, line) for one function of `nvdisasm -g` output."""
    amap = {}
    cur = None
    inside = False
    for ln in open(path):
        if ln.startswith("//---------------------"):
            inside = (".text." + func + " ") in ln or ln.rstrip().endswith(".text." + func + " --------------------------")
            if ".text." + func in ln:
                inside = True
            elif inside and ".text." in ln:
                inside = False
            continue
        if not inside:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and cur:
            amap[int(m.group(1), 16)] = cur
    return amap


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("sass_g")
    ap.add_argument("func")
    ap.add_argument("ncu_csv")
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--src", default=os.path.join(os.path.dirname(__file__), "..",
                                                  "paper_2604_27210_b200", "csrc"))
    a = ap.parse_args()
    amap = parse_lineinfo(a.sass_g, a.func)
    rows = list(csv.reader(open(a.ncu_csv)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    by_line = collections.Counter()
    samp_line = collections.Counter()
    mix_line = collections.defaultdict(collections.Counter)
    tot = 0
    seen = set()
    base = None
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        try:
            addr = int(r[ix["Address"]], 16)
            if base is None:
                base = addr
            addr -= base
            ie = int(r[ix["Instructions Executed"]] or 0)
            s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        except ValueError:
            continue
        if addr in seen:
            continue
        seen.add(addr)
        key = amap.get(addr, ("?", 0))
        src = r[ix["Source"]].strip().split()
        op = src[1] if src and src[0].startswith("@") and len(src) > 1 else (src[0] if src else "")
        by_line[key] += ie
        samp_line[key] += s
        mix_line[key][op.split(".")[0]] += ie
        tot += ie
    S = sum(samp_line.values()) or 1
    cache = {}
    print("total warp instructions %d, samples %d" % (tot, S))
    for key, v in by_line.most_common(a.top):
        f, line = key
        if f not in cache:
            p = os.path.join(a.src, f)
            cache[f] = open(p).read().splitlines() if os.path.exists(p) else []
        text = cache[f][line - 1].strip()[:70] if 0 < line <= len(cache[f]) else ""
        mix = ",".join("%s:%d" % (k, 100 * c // max(v, 1)) for k, c in mix_line[key].most_common(4))
        print("%5.1f%% inst %5.1f%% smp  %s:%-5d %-70s [%s]" % (100 * v / tot, 100 * samp_line[key] / S,
                                                          f, line, text, mix))


if __name__ == "__main__":
    main()
