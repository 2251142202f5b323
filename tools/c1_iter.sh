#!/bin/bash
# C1 kernel iteration: pair-reduce parity, two bench lines, ncu full capture of the K2 kernel
set -u
TAG=${1:-c1}
timeout 600 python -m pytest tests/test_gpu_pair_tma.py tests/test_gpu_ops.py -x -q > gpurun_out/t_$TAG.log 2>&1; tail -2 gpurun_out/t_$TAG.log
for r in 1 2; do
timeout 300 python bench.py --workload c1 --no-cpu-baseline > gpurun_out/b_$TAG.json 2>gpurun_out/b_$TAG.log
python -c "
import json; d=json.loads(open('gpurun_out/b_$TAG.json').read().strip().splitlines()[-1]); r=d['roofline']; print('value', d['value'], 'ms/step', d['ms_per_step'], 'frac', r['frac'], 'avg_launch_ms', r['avg_launch_ms'])"
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:reduce_tma -s 3 -c 1 -o gpurun_out/$TAG python bench.py --workload c1 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_$TAG.log 2>&1; grep -E "ERROR|Report" gpurun_out/ncu_$TAG.log
