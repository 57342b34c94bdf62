#!/bin/bash
# ncu --set full (source counters) of the LBR kernels on a 10M strided C4 sample,
# plus the SASS source pages of the far-low and normalize passes.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-lbr}
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:${KREGEX:-k_lbr_far_low_fast}" -c ${NCU_C:-1} \
  -o gpurun_out/prof_${TAG} python bench.py --rows 10000000 --steps 1 --warmup 0 --no-e2e --no-cpu --no-kernel-timing > gpurun_out/ncu_${TAG}.log 2>&1
tail -1 gpurun_out/ncu_${TAG}.log
for k in ${KLIST:-k_lbr_far_low_fast}; do
  ncu -i gpurun_out/prof_${TAG}.ncu-rep --page source --csv --print-source sass --kernel-name-base mangled -k regex:$k > gpurun_out/src_${TAG}_$k.csv 2>/dev/null
done
python tools/ncu_summary.py gpurun_out/prof_${TAG}.ncu-rep > gpurun_out/sum_${TAG}.txt 2>&1 || true
