set -u
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_kway_candidates" -s 3 -c 1 -o gpurun_out/r2_q6_kcand python bench.py --workload q6 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_ncu_kway.log 2>&1
