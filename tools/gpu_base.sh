cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for w in c2 c3 c1 c4; do
  timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu --no-kernel-timing 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$w', '%.3f Gq/s'%(d['value']/1e9), '%.3f ms'%d['ms_per_step'], 'frac %.3f'%d['roofline']['frac'], d.get('parity'))"
done
