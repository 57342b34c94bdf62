#!/bin/bash
# e2e (host-buffer C-ABI calls) A/B of variants/lib_*.so on $WLS
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for w in ${WLS:-c1 c2 c3}; do for rep in 1 2; do for lib in variants/lib_*.so; do
  n=$(basename $lib .so)
  FV_LIB=$PWD/$lib timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu --no-kernel-timing 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$w', '$n', 'dev %.3f'%(d['value']/1e9), 'e2e %.3f'%(d['e2e']['value']/1e9), 'ms %.2f'%d['e2e']['ms_per_step'])"
done; done; done
