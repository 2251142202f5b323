# pipelined segment bounds in the K12 row loop: parity (strict JIT) + A/B on Q6 / C5, x resident CTAs
set -u
rm -rf gpurun_out/pipe; mkdir -p gpurun_out/pipe
timeout 1200 python -m pytest tests/test_gpu_exprs.py tests/test_gpu_plans.py tests/test_gpu_configs.py tests/test_c5.py tests/test_gpu_queries.py tests/test_gpu_determinism.py tests/test_gpu_graphs.py -x -q --timeout 300 > gpurun_out/pipe/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/pipe/pytest.log
for rep in 1 2; do
  for cfg in "1 3" "0 3" "1 4" "0 4"; do
    set -- $cfg
    for wl in q6 c5; do
      RQ_JIT_PIPE=$1 RQ_JIT_MINB=$2 timeout 600 python bench.py --workload $wl --no-cpu-baseline --no-e2e --steps 30 > gpurun_out/pipe/p$1_m$2_${wl}_r$rep.json 2> /dev/null
    done
  done
done
timeout 600 python bench.py --workload q1 --no-cpu-baseline --no-e2e > gpurun_out/pipe/q1.json 2> gpurun_out/pipe/q1.log
tail -3 gpurun_out/pipe/pytest.log
