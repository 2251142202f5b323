# candidate pass, four run ends per thread: parity + Q6 / C5 bench + warm launch lists
set -u
rm -rf gpurun_out/cand; mkdir -p gpurun_out/cand
timeout 1200 python -m pytest tests/test_gpu_exprs.py tests/test_gpu_plans.py tests/test_gpu_configs.py tests/test_c5.py tests/test_gpu_queries.py tests/test_gpu_determinism.py tests/test_gpu_graphs.py tests/test_gpu_sharded.py -x -q --timeout 300 > gpurun_out/cand/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/cand/pytest.log
for wl in q6 c5 q1; do
  timeout 600 python bench.py --workload $wl --no-cpu-baseline --no-e2e --steps 30 > gpurun_out/cand/bench_$wl.json 2> gpurun_out/cand/bench_$wl.log
done
for wl in q6 c5; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/cand/warm_$wl.csv python bench.py --workload $wl --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
tail -3 gpurun_out/cand/pytest.log
