# last refresh of the lines the final K12 change moved (Q6, C5) + the GPU suite + smoke on HEAD
set -u
O=gpurun_out/final5; rm -rf $O; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
for wl in q6 c5 c2; do timeout 900 python bench.py --workload $wl > $O/bench_$wl.json 2> $O/bench_$wl.log; done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv --log-file $O/warm_q6.csv python bench.py --workload q6 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
tail -2 $O/pytest_gpu.log
