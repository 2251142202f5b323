#!/bin/bash
# K12 L2-prefetch A/B on a short-segment (Q6) and a long-segment (Q1) plan
for r in 1 2; do for pf in 0 1; do for w in q6 q1; do
RQ_JIT_PF=$pf timeout 300 python bench.py --workload $w --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; k=d['kernel_times_ms']['xg_rows']
print('pf $pf $w', 'ms/step %.4f'%d['ms_per_step'], 'frac %.3f'%r['frac'], 'xg_rows %.4f'%(k['ms']/k['count']))"
done; done; done
