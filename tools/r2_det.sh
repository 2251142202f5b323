# deterministic K10 f64 flushes: tests; Q1 / C3 / Q6 / C5 bench lines; row-kernel occupancy A/B on Q6 / C5
set -u
rm -rf gpurun_out/det; mkdir -p gpurun_out/det
timeout 900 python -m pytest tests/test_gpu_determinism.py tests/test_gpu_graphs.py tests/test_gpu_boundary.py tests/test_gpu_groupby.py -q --timeout 300 > gpurun_out/det/pytest_new.log 2>&1; echo "pytest exit $?" >> gpurun_out/det/pytest_new.log
timeout 1200 python -m pytest tests/test_gpu_exprs.py tests/test_gpu_plans.py tests/test_gpu_configs.py tests/test_c5.py tests/test_gpu_queries.py tests/test_gpu_ops.py -x -q --timeout 300 > gpurun_out/det/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/det/pytest.log
for wl in q1 c3 q6 c5; do
  timeout 600 python bench.py --workload $wl --no-cpu-baseline > gpurun_out/det/bench_$wl.json 2> gpurun_out/det/bench_$wl.log
done
for mb in 4 6; do
  for wl in q6 c5; do
    RQ_JIT_MINB=$mb timeout 600 python bench.py --workload $wl --no-cpu-baseline --no-e2e > gpurun_out/det/minb${mb}_$wl.json 2> gpurun_out/det/minb${mb}_$wl.log
  done
done
tail -3 gpurun_out/det/pytest_new.log gpurun_out/det/pytest.log
