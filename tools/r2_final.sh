# round-2 final: every bench line (e2e + cpu baseline), reference arm, ncu full captures of the dominant kernels
set -u
mkdir -p gpurun_out/final
for wl in c2 c1 c3 q1 q6 c5; do
  timeout 900 python bench.py --workload $wl > gpurun_out/final/bench_$wl.json 2> gpurun_out/final/bench_$wl.log
done
timeout 900 python bench.py --workload c2 --variant narrow > gpurun_out/final/bench_c2_narrow.json 2> gpurun_out/final/bench_c2_narrow.log
for wl in c2 c1 c3 q1 q6 c5; do
  timeout 600 python bench.py --impl reference --workload $wl --steps 3 --warmup 3 > gpurun_out/final/ref_$wl.json 2> gpurun_out/final/ref_$wl.log
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_points_filtered_reduce_tma" -s 3 -c 1 -o gpurun_out/final/c2_tma python bench.py --workload c2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python profiles/ncu_summarize.py gpurun_out/final/c2_tma.ncu-rep > gpurun_out/final/c2_tma_ncu_summary.txt 2>&1; python profiles/ncu_lines.py gpurun_out/final/c2_tma.ncu-rep 40 > gpurun_out/final/c2_tma_ncu_lines.txt 2>&1; rm -f gpurun_out/final/c2_tma.ncu-rep
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_pair_reduce_tma" -s 3 -c 1 -o gpurun_out/final/c1_k2 python bench.py --workload c1 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python profiles/ncu_summarize.py gpurun_out/final/c1_k2.ncu-rep > gpurun_out/final/c1_k2_ncu_summary.txt 2>&1; python profiles/ncu_lines.py gpurun_out/final/c1_k2.ncu-rep 40 > gpurun_out/final/c1_k2_ncu_lines.txt 2>&1; rm -f gpurun_out/final/c1_k2.ncu-rep
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"xg_kernel" -s 3 -c 1 -o gpurun_out/final/q1_xg python bench.py --workload q1 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python profiles/ncu_summarize.py gpurun_out/final/q1_xg.ncu-rep > gpurun_out/final/q1_xg_ncu_summary.txt 2>&1; python profiles/ncu_lines.py gpurun_out/final/q1_xg.ncu-rep 40 > gpurun_out/final/q1_xg_ncu_lines.txt 2>&1; rm -f gpurun_out/final/q1_xg.ncu-rep
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_kway_candidates|xg_kernel" -s 6 -c 2 -o gpurun_out/final/q6_kway python bench.py --workload q6 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python profiles/ncu_summarize.py gpurun_out/final/q6_kway.ncu-rep > gpurun_out/final/q6_kway_ncu_summary.txt 2>&1; python profiles/ncu_lines.py gpurun_out/final/q6_kway.ncu-rep 40 > gpurun_out/final/q6_kway_ncu_lines.txt 2>&1; rm -f gpurun_out/final/q6_kway.ncu-rep
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"xg_kernel|k_gk_items|k_gk_rle" -s 6 -c 3 -o gpurun_out/final/c3_group python bench.py --workload c3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python profiles/ncu_summarize.py gpurun_out/final/c3_group.ncu-rep > gpurun_out/final/c3_group_ncu_summary.txt 2>&1; python profiles/ncu_lines.py gpurun_out/final/c3_group.ncu-rep 40 > gpurun_out/final/c3_group_ncu_lines.txt 2>&1; rm -f gpurun_out/final/c3_group.ncu-rep
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/final/launches_c2_narrow.csv python bench.py --workload c2 --variant narrow --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls gpurun_out/final
