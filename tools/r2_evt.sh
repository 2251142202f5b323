set -u
rm -rf gpurun_out/evt; mkdir -p gpurun_out/evt
timeout 900 python -m pytest tests/test_gpu_graphs.py tests/test_gpu_determinism.py tests/test_gpu_exprs.py tests/test_gpu_configs.py -x -q --timeout 300 > gpurun_out/evt/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/evt/pytest.log
for wl in q6 c5 q1; do
  timeout 600 python bench.py --workload $wl --no-cpu-baseline --no-e2e > gpurun_out/evt/bench_$wl.json 2> gpurun_out/evt/bench_$wl.log
done
tail -3 gpurun_out/evt/pytest.log
