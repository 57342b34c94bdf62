#!/bin/bash
# A/B of variants/lib_*.so (tools/build_variants.py) on the workloads in $WLS,
# after the GPU parity subset in $TESTK.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_price_iv.py -x -q -k "${TESTK:-halley or c2 or exception or host or first or odd or price_iv or round}" 2>&1 | tail -2
for w in ${WLS:-c1 c5 c4}; do for rep in 1 2; do BENCH_ARGS="--workload $w --no-kernel-timing" bash tools/bench_variants.sh | sed "s/^/$w /"; done; done
