# skew tests + ncu --set full of the k-way placement kernel (Q6 / C5)
set -u
O=gpurun_out/sel; rm -rf $O; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_skew.py -q --timeout 600 > $O/pytest_skew.log 2>&1; echo "exit $?" >> $O/pytest_skew.log
for wl in c5 q6; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_kway_select" -s 3 -c 1 -o $O/sel_$wl python bench.py --workload $wl --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  python profiles/ncu_summarize.py $O/sel_$wl.ncu-rep > $O/sel_${wl}_summary.txt 2>&1
  python profiles/ncu_lines.py $O/sel_$wl.ncu-rep 40 > $O/sel_${wl}_lines.txt 2>&1
  rm -f $O/sel_$wl.ncu-rep
done
tail -3 $O/pytest_skew.log
