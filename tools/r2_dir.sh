# rank directories + profile filter: parity suites touching K12, Q6 / C5 / Q1 bench lines, warm launch lists, host split
set -u
rm -rf gpurun_out/dir; mkdir -p gpurun_out/dir
timeout 1800 python -m pytest tests/test_gpu_exprs.py tests/test_gpu_plans.py tests/test_gpu_configs.py tests/test_c5.py tests/test_gpu_queries.py tests/test_gpu_sharded.py -x -q > gpurun_out/dir/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/dir/pytest.log
for wl in q6 c5 q1 c3; do
  timeout 900 python bench.py --workload $wl --no-cpu-baseline > gpurun_out/dir/bench_$wl.json 2> gpurun_out/dir/bench_$wl.log
done
for wl in q6 c5; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/dir/warm_$wl.csv python bench.py --workload $wl --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  timeout 600 python tools/q_host.py $wl 50 > gpurun_out/dir/host_$wl.txt 2>&1
done
tail -3 gpurun_out/dir/pytest.log
