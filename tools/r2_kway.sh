# k-way segment builder: parity suites touching group_aggregate_exprs, then Q6 / C5 / Q1 bench lines + launch lists
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_exprs.py tests/test_gpu_plans.py tests/test_gpu_configs.py tests/test_c5.py tests/test_gpu_queries.py tests/test_gpu_sharded.py -x -q > gpurun_out/r2_kway_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2_kway_pytest.log
for wl in q6 c5 q1; do
  timeout 900 python bench.py --workload $wl --no-cpu-baseline > gpurun_out/r2_kway_$wl.json 2> gpurun_out/r2_kway_$wl.log
done
for wl in q6 c5; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_$wl.csv python bench.py --workload $wl --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
tail -3 gpurun_out/r2_kway_pytest.log
