#!/bin/bash
# A/B of variants/lib_*.so on $WLS (default c3 c2 rt), after the pricing /
# Halley parity subset on the default build.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_price_iv.py -x -q -k "${TESTK:-price or greeks or halley or c2 or c3 or golden}" 2>&1 | tail -2
for w in ${WLS:-c3 c2 rt}; do for rep in 1 2; do BENCH_ARGS="--workload $w --no-kernel-timing" bash tools/bench_variants.sh | sed "s/^/$w /"; done; done
