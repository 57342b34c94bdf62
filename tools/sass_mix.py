#!/usr/bin/env python3
"""Dynamic SASS instruction mix of one kernel from an ncu report's source page.

    ncu -i rep --page source --csv --print-source sass -k regex:NAME > k.csv
    python tools/sass_mix.py k.csv [--top 40]

Prints warp-level executed instructions by opcode (and by opcode class),
the share of FP64 instructions, and the hottest instructions with their
stall samples."""
import csv
import re
import sys
from collections import Counter, defaultdict

FP64 = {"DFMA", "DADD", "DMUL", "DSETP", "DMNMX", "DSET"}


def main():
    path = sys.argv[1]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 40
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    h = rows[hdr]
    ci = h.index("Instructions Executed")
    cs = h.index("Source")
    cst = h.index("Warp Stall Sampling (All Samples)")
    ct = h.index("Thread Instructions Executed")
    by_op = Counter()
    thr_op = Counter()
    stall_op = Counter()
    insts = []
    seen = set()
    for r in rows[hdr + 1:]:
        if len(r) <= ci:
            continue
        if r[0] in seen:           # the source page can list a kernel's SASS twice
            continue
        seen.add(r[0])
        try:
            n = int(r[ci]); nt = int(r[ct]); st = int(r[cst] or 0)
        except ValueError:
            continue
        src = r[cs].strip()
        m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[\w.]+)?", src)
        op = m.group(2) if m else src.split()[0]
        by_op[op] += n
        thr_op[op] += nt
        stall_op[op] += st
        insts.append((n, st, r[0], src))
    tot = sum(by_op.values())
    tot_st = sum(stall_op.values()) or 1
    fp = sum(v for k, v in by_op.items() if k in FP64)
    print(f"warp instructions {tot:,}; FP64 {fp:,} ({100.0 * fp / tot:.1f} %)")
    print(f"{'opcode':12s} {'warp inst':>14s} {'share':>7s} {'lanes':>6s} {'stall%':>7s}")
    for op, v in by_op.most_common(45):
        print(f"{op:12s} {v:14,d} {100.0 * v / tot:6.2f}% {thr_op[op] / max(v, 1):6.1f} {100.0 * stall_op[op] / tot_st:6.2f}%")
    print("\nhottest instructions (warp inst, stall samples):")
    for n, st, addr, src in sorted(insts, key=lambda x: -x[1])[:top]:
        print(f"{n:12,d} {st:7d}  {src}")


if __name__ == "__main__":
    main()
