#!/bin/bash
# FP64 instruction counts per workload call (ncu, serialised): thread-level
# DADD / DMUL / DFMA with the predicate on (= lanes that did the work), warp-level
# FP64-pipe instructions, all instructions, time.  -> gpurun_out/fp64_<w>.csv
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
M=gpu__time_duration.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__inst_executed_pipe_fp64.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active
for spec in c4:k_lbr c1:k_lbr c5:k_lbr c2:k_halley c3:k_price_greeks rt:k_price\|k_halley; do
  w=${spec%%:*}; k=${spec#*:}
  ROWS=""; [ $w = c4 ] && ROWS="--rows 10000000"
  timeout 900 ncu --metrics $M --clock-control none -k regex:$k --csv --log-file gpurun_out/fp64_$w.csv \
    python bench.py --workload $w $ROWS --steps 1 --warmup 0 --no-e2e --no-cpu --no-kernel-timing > /dev/null 2>&1
done
ls -la gpurun_out/fp64_*.csv
