set -x
for ov in 0 1; do ZK_DIST_OVERLAP=$ov timeout 1500 python bench.py --local-ranks 4 --steps 2 --warmup 1 2>/dev/null | python -c "
import sys, json; d = json.loads(sys.stdin.read().strip().splitlines()[-1]); print('overlap=$ov', round(d['value']), 'GB/s', round(d['bicgstab']['ms_per_iteration'], 3), 'ms/it', d['bicgstab']['iters'], 'it')"; done
