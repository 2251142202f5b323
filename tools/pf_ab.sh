#!/bin/bash
# K12 row-kernel L2 prefetch A/B (RQ_JIT_PF = windows ahead; 0 = off)
timeout 900 python -m pytest tests/test_gpu_exprs.py tests/test_gpu_queries.py tests/test_c5.py -x -q 2>&1 | tail -1
for pf in 0 2 1 4; do
for w in q1 c3; do
RQ_JIT_PF=$pf timeout 300 python bench.py --workload $w --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; k=d['kernel_times_ms']
print('pf $pf $w', 'ms/step %.4f'%d['ms_per_step'], 'frac %.3f'%r['frac'], 'xg_rows %.4f'%(k.get('xg_rows',{'ms':0,'count':1})['ms']/k.get('xg_rows',{'count':1})['count']))"
done; done
