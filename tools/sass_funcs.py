#!/usr/bin/env python3
"""Inclusive per-function profile of one kernel from an ncu SASS source page
and `nvdisasm -gi` inline line info: every SASS address is charged to every
source function on its inline chain (innermost to the kernel), so the table
reads like a call-tree profile ("fx_erfc_warp 31 % of the warp instructions,
of which fx_erfc_tail 12 %").

    nvdisasm -gi -c fv_kernels.sm_100a.cubin > all_gi.sass
    ncu -i rep.ncu-rep --page source --csv --print-source sass \
        --kernel-name-base mangled -k regex:<name> > k.csv
    python tools/sass_funcs.py all_gi.sass <mangled-name> k.csv [--top 50]
"""
import argparse
import collections
import csv
import os
import re

FUNC_RE = re.compile(r"^\s*(?:template\s*<[^>]*>\s*)?(?:FV_HD|FV_HDM|__device__|__global__|static|inline)[^;{]*?\b(\w+)\s*\(")


def func_starts(path):
    """[(line, name)] of function definitions in a source file (heuristic)."""
    out = []
    try:
        lines = open(path).read().splitlines()
    except OSError:
        return out
    for i, ln in enumerate(lines, 1):
        m = FUNC_RE.match(ln)
        if m and not ln.rstrip().endswith(";"):
            out.append((i, m.group(1)))
    return out


def parse_chains(path, func):
    """address -> [(file, line), ...] innermost first, for one function."""
    # A group of `//## File` records precedes each run of instructions: one
    # record per inline level, innermost first, the last one (no "inlined
    # at") being the kernel's own line.
    amap = {}
    chain = []
    pending = []
    inside = False
    for ln in open(path):
        if ".text." in ln and ("//-----" in ln or ".section" in ln):
            inside = re.search(r"\.text\.%s\b" % re.escape(func), ln) is not None
            continue
        if not inside:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            pending.append((os.path.basename(m.group(1)), int(m.group(2))))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m:
            if pending:
                chain, pending = pending, []
            if chain:
                amap[int(m.group(1), 16)] = list(chain)
    return amap


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("sass_gi")
    ap.add_argument("func")
    ap.add_argument("ncu_csv")
    ap.add_argument("--top", type=int, default=50)
    ap.add_argument("--src", default=os.path.join(os.path.dirname(os.path.abspath(__file__)), "..",
                                                  "paper_2604_27210_b200", "csrc"))
    a = ap.parse_args()
    starts = {}

    def fname(f, line):
        if f not in starts:
            starts[f] = func_starts(os.path.join(a.src, f))
        best = f
        for l0, n in starts[f]:
            if l0 <= line:
                best = n
            else:
                break
        return best

    amap = parse_chains(a.sass_gi, a.func)
    rows = list(csv.reader(open(a.ncu_csv)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    incl = collections.Counter()
    excl = collections.Counter()
    fp64 = collections.Counter()
    samp = collections.Counter()
    tot = tot_s = 0
    base = None
    seen = set()
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
        src = r[ix["Source"]].strip().split()
        op = src[1] if src and src[0].startswith("@") and len(src) > 1 else (src[0] if src else "")
        isf = op.split(".")[0] in ("DFMA", "DADD", "DMUL", "DSETP", "DMNMX")
        chain = amap.get(addr, [("?", 0)])
        names = []
        for f, l in chain:
            n = fname(f, l)
            if n not in names:
                names.append(n)
        for n in names:
            incl[n] += ie
            samp[n] += s
            if isf:
                fp64[n] += ie
        excl[names[0]] += ie
        tot += ie
        tot_s += s
    print("total warp instructions %d, stall samples %d" % (tot, tot_s))
    print("%-28s %7s %7s %7s %7s" % ("function", "incl%", "excl%", "fp64%", "smp%"))
    for n, v in incl.most_common(a.top):
        print("%-28s %6.1f%% %6.1f%% %6.1f%% %6.1f%%" % (n[:28], 100 * v / tot, 100 * excl[n] / tot,
                                                       100 * fp64[n] / max(v, 1), 100 * samp[n] / max(tot_s, 1)))


if __name__ == "__main__":
    main()
