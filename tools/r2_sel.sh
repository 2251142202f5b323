set -u
rm -rf gpurun_out/sel; mkdir -p gpurun_out/sel
timeout 900 python -m pytest tests/test_gpu_exprs.py tests/test_gpu_configs.py tests/test_c5.py tests/test_gpu_queries.py tests/test_gpu_graphs.py tests/test_gpu_determinism.py -x -q --timeout 300 > gpurun_out/sel/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/sel/pytest.log
for wl in q6 c5; do
  timeout 600 python bench.py --workload $wl --no-cpu-baseline --no-e2e > gpurun_out/sel/bench_$wl.json 2> gpurun_out/sel/bench_$wl.log
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/sel/warm_$wl.csv python bench.py --workload $wl --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_kway_candidates" -s 3 -c 1 -o gpurun_out/sel/c5_cand python bench.py --workload c5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python profiles/ncu_summarize.py gpurun_out/sel/c5_cand.ncu-rep > gpurun_out/sel/c5_cand_summary.txt 2>&1
python profiles/ncu_lines.py gpurun_out/sel/c5_cand.ncu-rep 30 > gpurun_out/sel/c5_cand_lines.txt 2>&1
ncu -i gpurun_out/sel/c5_cand.ncu-rep --page details --csv > gpurun_out/sel/c5_cand_details.csv 2>&1
rm -f gpurun_out/sel/c5_cand.ncu-rep
tail -3 gpurun_out/sel/pytest.log
