#!/bin/bash
# Time every variants/lib_*.so on the C4 bench (device-resident), one line each.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for lib in variants/lib_*.so; do
  n=$(basename $lib .so)
  FV_LIB=$PWD/$lib timeout 300 python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu ${BENCH_ARGS:-} 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$n', '%.3f Gq/s'%(d['value']/1e9), '%.2f ms'%d['ms_per_step'], 'frac %.3f'%d['roofline']['frac'])"
done
