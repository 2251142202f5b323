# re-entry check of HEAD: GPU suite, smoke, every bench line
set -u
O=gpurun_out/reentry
rm -rf $O; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
for wl in c2 c1 q1 q6 c5 c3; do
  timeout 600 python bench.py --workload $wl > $O/bench_$wl.json 2> $O/bench_$wl.log
done
tail -3 $O/pytest_gpu.log
