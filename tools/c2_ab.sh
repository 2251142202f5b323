#!/bin/bash
# C2 A/B on one box: alternating bench lines of the in-tree build and of $1 (a .so)
for r in 1 2 3; do
for lib in "" "$1"; do
RQ_LIB_PATH=$lib timeout 300 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('${lib:-tree}', 'ms/step %.4f'%d['ms_per_step'], 'frac %.3f'%r['frac'], 'kernel_ms %.4f'%r['avg_launch_ms'])"
done
done
