#!/bin/bash
# ncu launch list (per-kernel duration, serialised) of one workload call:
#   W=c1 TAG=x tools/gpu_launches.sh
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-l}
W=${W:-c1}
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv \
  --log-file gpurun_out/launches_${TAG}_$W.csv python bench.py --workload $W ${ROWS:+--rows $ROWS} --steps 1 --warmup 0 --no-e2e --no-cpu --no-kernel-timing > /dev/null 2>&1
python - <<PY
import csv, collections
rows = list(csv.reader(open("gpurun_out/launches_${TAG}_$W.csv")))
hdr = None
out = []
for r in rows:
    if r and r[0] == "ID": hdr = r; continue
    if hdr and len(r) == len(hdr): out.append(dict(zip(hdr, r)))
ids = collections.OrderedDict()
for d in out:
    ids.setdefault(d["ID"], {"name": d["Kernel Name"][:60]})[d["Metric Name"]] = d["Metric Value"]
for i, v in list(ids.items())[-24:]:
    print(i, v["name"], v.get("gpu__time_duration.sum"), v.get("launch__grid_size"), v.get("sm__warps_active.avg.pct_of_peak_sustained_active"))
PY
