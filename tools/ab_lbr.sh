cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "lbr or c1 or c4 or c5 or host" 2>&1 | tail -2
for w in c1 c5 c4; do for rep in 1 2; do BENCH_ARGS="--workload $w --no-kernel-timing" bash tools/bench_variants.sh | sed "s/^/$w /"; done; done
