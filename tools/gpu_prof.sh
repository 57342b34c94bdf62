#!/bin/bash
# Targeted ncu --set full captures (source counters) of named kernels on one
# workload:  W=c2 KREGEX=k_halley NCU_C=5 TAG=x tools/gpu_prof.sh
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-p}
W=${W:-c2}
if [ -n "${PRE:-}" ]; then bash -c "$PRE"; fi
timeout ${TMO:-900} ncu --set full --clock-control none --import-source on -k "regex:${KREGEX:-k_halley}" -c ${NCU_C:-5} \
  -o gpurun_out/prof_${TAG} python bench.py --workload $W ${ROWS:+--rows $ROWS} --steps 1 --warmup 0 --no-e2e --no-cpu --no-kernel-timing \
  > gpurun_out/ncu_${TAG}.log 2>&1
tail -2 gpurun_out/ncu_${TAG}.log
