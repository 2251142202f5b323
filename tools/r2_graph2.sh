# determinism + graphs + warp-per-segment outliers + warp-range group folds: tests, Q6 / C5 / Q1 bench, warm lists
set -u
rm -rf gpurun_out/graph2; mkdir -p gpurun_out/graph2
timeout 900 python -m pytest tests/test_gpu_graphs.py tests/test_gpu_determinism.py tests/test_gpu_boundary.py -q --timeout 300 > gpurun_out/graph2/pytest_new.log 2>&1; echo "pytest exit $?" >> gpurun_out/graph2/pytest_new.log
timeout 1200 python -m pytest tests/test_gpu_exprs.py tests/test_gpu_plans.py tests/test_gpu_configs.py tests/test_c5.py tests/test_gpu_queries.py tests/test_gpu_groupby.py -x -q --timeout 300 > gpurun_out/graph2/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/graph2/pytest.log
for wl in q6 c5 q1; do
  timeout 600 python bench.py --workload $wl --no-cpu-baseline > gpurun_out/graph2/bench_$wl.json 2> gpurun_out/graph2/bench_$wl.log
done
for wl in q6 c5; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/graph2/warm_$wl.csv python bench.py --workload $wl --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
tail -3 gpurun_out/graph2/pytest_new.log gpurun_out/graph2/pytest.log
