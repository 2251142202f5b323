#!/bin/bash
# K12 iteration: expression parity tests, q1/q6/c5 bench lines, ncu of the row kernel (q1)
set -u
TAG=${1:-x}
timeout 900 python -m pytest tests/test_gpu_exprs.py tests/test_gpu_queries.py tests/test_c5.py tests/test_gpu_groupby.py tests/test_gpu_plans.py tests/test_gpu_encode.py -x -q > gpurun_out/t_$TAG.log 2>&1; tail -2 gpurun_out/t_$TAG.log
for w in q1 q6 c5; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/b_${TAG}_$w.json 2> gpurun_out/b_${TAG}_$w.log
  python -c "
import json; d=json.loads(open('gpurun_out/b_${TAG}_$w.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$w', 'value %.3g'%d['value'], 'ms/step %.3f'%d['ms_per_step'], 'frac %.3f'%r['frac'], 'tag_ms %.3f'%r['avg_launch_ms'], 'chain_ms %.3f'%d['chain_ms_per_step'])" || tail -3 gpurun_out/b_${TAG}_$w.log
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"xg_kernel|k_xg_rows" -c 1 -o gpurun_out/${TAG}_q1rows python bench.py --workload q1 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_${TAG}.log 2>&1; grep -E "ERROR|Report" gpurun_out/ncu_${TAG}.log
