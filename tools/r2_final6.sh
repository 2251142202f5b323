# final C2 refresh after the producer-side predicate flags: bench line, ncu --set full, launch list
set -u
O=gpurun_out/final6; rm -rf $O; mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench_c2.json 2> $O/bench_c2.log
timeout 900 python bench.py --workload c2 --variant narrow > $O/bench_c2_narrow.json 2> $O/bench_c2_narrow.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_points_filtered_reduce_tma" -s 3 -c 1 -o $O/c2_tma python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python profiles/ncu_summarize.py $O/c2_tma.ncu-rep > $O/c2_tma_ncu_summary.txt 2>&1
python profiles/ncu_lines.py $O/c2_tma.ncu-rep 40 > $O/c2_tma_ncu_lines.txt 2>&1
rm -f $O/c2_tma.ncu-rep
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls $O
