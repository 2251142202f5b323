# prepared query plans (Python args marshalled once): parity, Q6 / C5 / Q1 bench; Q1 chain launch list
set -u
rm -rf gpurun_out/prep; mkdir -p gpurun_out/prep
timeout 1200 python -m pytest tests/test_gpu_exprs.py tests/test_gpu_plans.py tests/test_gpu_configs.py tests/test_c5.py tests/test_gpu_queries.py tests/test_gpu_determinism.py tests/test_gpu_graphs.py tests/test_gpu_sharded.py -x -q --timeout 300 > gpurun_out/prep/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/prep/pytest.log
for wl in q6 c5 q1; do
  timeout 600 python bench.py --workload $wl --no-cpu-baseline > gpurun_out/prep/bench_$wl.json 2> gpurun_out/prep/bench_$wl.log
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prep/q1_chain.csv python bench.py --workload q1 --path chain --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/traffic_summary.py gpurun_out/prep/q1_chain.csv > gpurun_out/prep/q1_chain_summary.txt 2>&1 || true
tail -3 gpurun_out/prep/pytest.log
