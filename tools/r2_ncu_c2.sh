set -u
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_points_filtered_reduce_tma" -s 3 -c 1 -o gpurun_out/r2_c2_full python bench.py --workload c2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_ncu_c2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_pair_reduce_tma" -s 3 -c 1 -o gpurun_out/r2_c1_full python bench.py --workload c1 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_ncu_c1.log 2>&1
