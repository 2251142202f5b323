# round-2 final refresh (re-entry session, after the k-way / tail / prepared-call changes):
# GPU suite + smoke, every bench line, reference arm for the scalar workloads, ncu of the
# dominant kernels that changed, launch list of the default command, warm Q6 / C5 lists, C3 at 10B
set -u
O=gpurun_out/final4
rm -rf $O; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
for wl in c2 c1 c3 q1 q6 c5; do
  timeout 900 python bench.py --workload $wl > $O/bench_$wl.json 2> $O/bench_$wl.log
done
timeout 900 python bench.py --workload c2 --variant narrow > $O/bench_c2_narrow.json 2> $O/bench_c2_narrow.log
for wl in c2 c1; do
  timeout 600 python bench.py --impl reference --workload $wl --steps 3 --warmup 3 > $O/ref_$wl.json 2> $O/ref_$wl.log
done
ncu_full() {  # name, kernel regex, skip, count, bench args...
  local name=$1 rx=$2 s=$3 c=$4; shift 4
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$rx" -s $s -c $c -o $O/$name python bench.py "$@" --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  python profiles/ncu_summarize.py $O/$name.ncu-rep > $O/${name}_ncu_summary.txt 2>&1
  python profiles/ncu_lines.py $O/$name.ncu-rep 40 > $O/${name}_ncu_lines.txt 2>&1
  rm -f $O/$name.ncu-rep
}
ncu_full c5_kway "k_kway_candidates|k_kway_select|xg_kernel|k_xg_tail" 12 4 --workload c5
ncu_full q6_kway "k_kway_candidates|k_kway_select|xg_kernel" 9 3 --workload q6
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
for wl in q6 c5; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv --log-file $O/warm_$wl.csv python bench.py --workload $wl --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
timeout 2000 python bench.py --workload c3 --rows 10000000000 --steps 5 > $O/bench_c3_10b.json 2> $O/bench_c3_10b.log
ls $O
tail -2 $O/pytest_gpu.log
