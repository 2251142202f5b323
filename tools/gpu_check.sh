#!/bin/bash
# One gpurun call: GPU parity suite, smoke, bench lines for every workload,
# and the ncu launch list of the default bench command.
# Usage (from this container):
#   gpurun --timeout 2400 -- 'bash tools/gpu_check.sh [workloads...]'
set -u
OUT=gpurun_out
mkdir -p $OUT
WL=${@:-c2 c1 c3 q6 q1 c5}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
for w in $WL; do
  timeout 600 python bench.py --workload $w > $OUT/bench_$w.json 2> $OUT/bench_$w.log; echo "bench $w exit $?" >> $OUT/bench_$w.log
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $OUT/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_c2.log 2>&1
for w in c2 c1 c3 q6 q1 c5; do timeout 300 python tools/host_breakdown.py $w 10 2>/dev/null | head -1; done > $OUT/host_split.txt
echo done
