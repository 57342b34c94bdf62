#!/bin/bash
# Full round run on one B200: GPU tests, smoke, the C4 bench line (with e2e +
# CPU baseline + parity of every row), the other workloads (same), the
# reference arm, the drop-in Python API end to end, an ncu launch list of the
# bench command, ncu DRAM traffic per workload, and ncu --set full captures of
# the LBR, Halley and price+Greeks kernels.  Outputs in gpurun_out/.
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-full}
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu_${TAG}.txt 2>&1
lscpu > gpurun_out/cpu_${TAG}.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/pytest_gpu_${TAG}.txt
tail -3 gpurun_out/pytest_gpu_${TAG}.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.txt 2>&1; tail -1 gpurun_out/smoke_${TAG}.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; tail -c 400 gpurun_out/bench_${TAG}.json; echo
for w in c1 c2 c3 c5 rt; do
  timeout 600 python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/bench_${TAG}_$w.json 2>> gpurun_out/bench_${TAG}.err
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_${TAG}_ref.json 2>> gpurun_out/bench_${TAG}.err; head -c 300 gpurun_out/bench_${TAG}_ref.json; echo
timeout 600 python tools/api_e2e.py 50000000 > gpurun_out/api_e2e_${TAG}.json 2>> gpurun_out/bench_${TAG}.err; cat gpurun_out/api_e2e_${TAG}.json | head -c 600; echo
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
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_price_greeks -c 1 -o gpurun_out/profg_${TAG} python bench.py --workload c3 --steps 1 --warmup 0 --no-e2e --no-cpu --no-kernel-timing > gpurun_out/ncug_${TAG}.log 2>&1
  tail -1 gpurun_out/ncug_${TAG}.log
fi
if [ "${SAN:-1}" = "1" ]; then
  for tool in memcheck racecheck synccheck initcheck; do
    timeout 1200 compute-sanitizer --tool $tool --error-exitcode 1 python tools/sanitize.py > gpurun_out/sanitize_${TAG}_$tool.log 2>&1
    echo "sanitize $tool rc=$? $(tail -1 gpurun_out/sanitize_${TAG}_$tool.log)"
  done
fi
timeout 600 python tools/chain_e2e.py 1000000 "price,iv,greeks" > gpurun_out/chain_e2e_${TAG}.json 2>> gpurun_out/bench_${TAG}.err
