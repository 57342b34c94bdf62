#!/bin/bash
# Full round run on one B200: GPU tests, smoke, the C4 bench line (with e2e +
# CPU baseline), the other workloads, the reference arm, an ncu launch list of
# the bench command, ncu DRAM traffic per workload, and an ncu --set full
# capture of the LBR kernels.  Outputs in gpurun_out/.
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-full}
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu_${TAG}.txt 2>&1
lscpu > gpurun_out/cpu_${TAG}.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/pytest_gpu_${TAG}.txt
tail -3 gpurun_out/pytest_gpu_${TAG}.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.txt 2>&1; tail -1 gpurun_out/smoke_${TAG}.txt
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; tail -c 600 gpurun_out/bench_${TAG}.json
for w in c1 c2 c3 c5 rt; do
  timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_${TAG}_$w.json 2>> gpurun_out/bench_${TAG}.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_${TAG}_ref.json 2>> gpurun_out/bench_${TAG}.err; cat gpurun_out/bench_${TAG}_ref.json | head -c 400; echo
if [ "${NCU:-1}" = "1" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
  M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
  for spec in c4:k_lbr c1:k_lbr c5:k_lbr c2:k_halley c3:k_price_greeks rt:k_price\|k_halley; do
    w=${spec%%:*}; k=${spec#*:}
    timeout 900 ncu --metrics $M --clock-control none -k regex:$k --csv --log-file gpurun_out/traffic_${TAG}_$w.csv python bench.py --workload $w --steps 1 --warmup 0 --no-e2e --no-cpu --no-kernel-timing > /dev/null 2>&1
  done
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lbr -c 7 -o gpurun_out/prof_${TAG} python bench.py --rows 10000000 --steps 1 --warmup 0 --no-e2e --no-cpu --no-kernel-timing > gpurun_out/ncu_${TAG}.log 2>&1
  tail -1 gpurun_out/ncu_${TAG}.log
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_halley -c 5 -o gpurun_out/profh_${TAG} python bench.py --workload c2 --steps 1 --warmup 0 --no-e2e --no-cpu --no-kernel-timing > gpurun_out/ncuh_${TAG}.log 2>&1
  tail -1 gpurun_out/ncuh_${TAG}.log
fi
