#!/bin/bash
# C3 iteration: group-by parity tests, c3 bench line, per-kernel traffic of one c3 step
set -u
TAG=${1:-x}
timeout 900 python -m pytest tests/test_gpu_groupby.py tests/test_gpu_queries.py tests/test_gpu_plans.py tests/test_c5.py tests/test_gpu_exprs.py -x -q > gpurun_out/t_$TAG.log 2>&1; tail -2 gpurun_out/t_$TAG.log
timeout 600 python bench.py --workload c3 --no-cpu-baseline > gpurun_out/b_${TAG}_c3.json 2> gpurun_out/b_${TAG}_c3.log
python -c "
import json; d=json.loads(open('gpurun_out/b_${TAG}_c3.json').read().strip().splitlines()[-1]); r=d['roofline']; print('c3', 'value %.3g'%d['value'], 'ms/step %.3f'%d['ms_per_step'], 'frac %.3f'%r['frac'], 'tag_ms %.3f'%r['avg_launch_ms'])" || tail -3 gpurun_out/b_${TAG}_c3.log
timeout 600 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/traffic_${TAG}_c3.csv python tools/ncu_query.py c3 > /dev/null 2>&1
python tools/traffic_summary.py gpurun_out/traffic_${TAG}_c3.csv > gpurun_out/traffic_${TAG}_c3.txt; head -6 gpurun_out/traffic_${TAG}_c3.txt
