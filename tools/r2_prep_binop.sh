set -u
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -2
for r in 1 2 3; do for wl in c2 c1; do
timeout 300 python bench.py --workload $wl --steps 20 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); r=d['roofline']; print('$wl', round(d['ms_per_step'],5), round(r['avg_launch_ms'],5), round(r['frac'],4), d['oracle_match'])"
done; done
