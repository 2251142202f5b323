# CUDA-graph replay of K12 plans (pieces around profiled regions), deterministic f64 folds, chunk-start table
set -u
rm -rf gpurun_out/graph; mkdir -p gpurun_out/graph
timeout 1800 python -m pytest tests/test_gpu_graphs.py tests/test_gpu_determinism.py -q > gpurun_out/graph/pytest_new.log 2>&1; echo "pytest exit $?" >> gpurun_out/graph/pytest_new.log
timeout 1800 python -m pytest tests/test_gpu_exprs.py tests/test_gpu_plans.py tests/test_gpu_configs.py tests/test_c5.py tests/test_gpu_queries.py tests/test_gpu_sharded.py tests/test_gpu_groupby.py -x -q > gpurun_out/graph/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/graph/pytest.log
for wl in q6 c5 q1; do
  timeout 900 python bench.py --workload $wl --no-cpu-baseline > gpurun_out/graph/bench_$wl.json 2> gpurun_out/graph/bench_$wl.log
  RQ_NO_GRAPH=1 timeout 900 python bench.py --workload $wl --no-cpu-baseline --no-e2e > gpurun_out/graph/nograph_$wl.json 2> gpurun_out/graph/nograph_$wl.log
done
for wl in q6 c5; do
  timeout 600 python tools/q_host.py $wl 50 > gpurun_out/graph/host_$wl.txt 2>&1
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/graph/warm_$wl.csv python bench.py --workload $wl --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
tail -3 gpurun_out/graph/pytest_new.log gpurun_out/graph/pytest.log
