#!/bin/bash
# Quick GPU iteration: GPU parity tests (LBR-focused subset unless FULL=1),
# a C4 bench line, and an ncu capture of the LBR kernels on a 10M strided sample.
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-q}
if [ "${FULL:-0}" = "1" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
else
  timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "${TESTK:-lbr or c1 or c4 or c5 or first}" 2>&1 | tail -8
fi
timeout 600 python bench.py --steps ${STEPS:-3} --warmup 1 ${BENCH_ARGS:---no-e2e --no-cpu} > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
python - <<'PY'
import json, os
tag = os.environ.get("TAG", "q")
try:
    d = json.loads(open(f"gpurun_out/bench_{tag}.json").read().strip().splitlines()[-1])
    print("BENCH value %.3f Gq/s  ms/step %.2f  fp64 frac %.3f  per_call %s" % (d["value"]/1e9, d["ms_per_step"], d["roofline"]["frac"], [round(x,2) for x in d["per_call_ms"]]))
    if d.get("e2e"): print("E2E %.3f Gq/s" % (d["e2e"]["value"]/1e9))
    if d.get("cpu_baseline"): print("CPU", d["cpu_baseline"])
except Exception as e:
    print("bench failed", e); print(open(f"gpurun_out/bench_{tag}.err").read()[-3000:])
PY
if [ "${NCU:-1}" = "1" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:${KREGEX:-k_lbr}" -c ${NCU_C:-4} -o gpurun_out/prof_${TAG} python bench.py --rows 10000000 --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu_${TAG}.log 2>&1
  tail -2 gpurun_out/ncu_${TAG}.log
fi
