cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for w in c1 c4; do
ROWS=""; [ $w = c4 ] && ROWS="--rows 10000000"
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__thread_inst_executed_per_inst_executed.ratio,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv -k regex:k_lbr \
  --log-file gpurun_out/lanes_$w.csv python bench.py --workload $w $ROWS --steps 1 --warmup 0 --no-e2e --no-cpu --no-kernel-timing > /dev/null 2>&1
python - <<PY
import csv, collections
rows=list(csv.reader(open("gpurun_out/lanes_$w.csv")))
hdr=None; d=collections.OrderedDict()
for r in rows:
    if r and r[0]=="ID": hdr=r; continue
    if hdr and len(r)==len(hdr):
        x=dict(zip(hdr,r)); d.setdefault(x["ID"],{"k":x["Kernel Name"][:34]})[x["Metric Name"].split("__")[1][:28]]=x["Metric Value"]
for i,v in list(d.items())[-9:]: print("$w", v)
PY
done
