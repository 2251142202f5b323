# round-2 refresh: parity subset, every bench line, reference arm, ncu launch lists
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_exprs.py tests/test_gpu_plans.py tests/test_gpu_configs.py tests/test_c5.py -x -q > gpurun_out/r2_refresh_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2_refresh_pytest.log
for wl in c2 c1 c3 q1 q6 c5; do
  timeout 900 python bench.py --workload $wl > gpurun_out/r2_bench_$wl.json 2> gpurun_out/r2_bench_$wl.log
done
timeout 900 python bench.py --workload c2 --variant narrow > gpurun_out/r2_bench_c2_narrow.json 2> gpurun_out/r2_bench_c2_narrow.log
timeout 600 python bench.py --impl reference > gpurun_out/r2_bench_ref_c2.json 2> gpurun_out/r2_bench_ref_c2.log
for wl in c2 c1 q6 c5; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_$wl.csv python bench.py --workload $wl --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_launches_c2_narrow.csv python bench.py --workload c2 --variant narrow --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
tail -3 gpurun_out/r2_refresh_pytest.log
