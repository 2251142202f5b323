# config-level parity + bench lines with full-table oracle gates (round 2)
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_configs.py -x -q > gpurun_out/r2_configs_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2_configs_pytest.log
for wl in c3 q1 q6 c5; do
  timeout 900 python bench.py --workload $wl > gpurun_out/r2_bench_$wl.json 2> gpurun_out/r2_bench_$wl.log
done
timeout 1800 python bench.py --workload c3 --rows 10000000000 --steps 5 > gpurun_out/r2_bench_c3_10b.json 2> gpurun_out/r2_bench_c3_10b.log
nvidia-smi --query-gpu=memory.used,memory.total --format=csv >> gpurun_out/r2_bench_c3_10b.log
tail -3 gpurun_out/r2_configs_pytest.log
