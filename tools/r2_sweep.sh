# C1 L sweep at 1B rows and C1 at its configured 10M rows; C3 at 10B after the round-2 changes
set -u
mkdir -p gpurun_out/sweep
for L in 16,24 64,96 1000,1500; do
  timeout 900 python bench.py --workload c1 --c1-runs $L --no-cpu-baseline > gpurun_out/sweep/c1_1b_${L/,/_}.json 2> gpurun_out/sweep/c1_1b_${L/,/_}.log
done
timeout 900 python bench.py --workload c1 --rows 10000000 > gpurun_out/sweep/c1_10m.json 2> gpurun_out/sweep/c1_10m.log
timeout 600 python bench.py --impl reference --workload c1 --rows 10000000 --steps 5 > gpurun_out/sweep/ref_c1_10m.json 2> gpurun_out/sweep/ref_c1_10m.log
timeout 2400 python bench.py --workload c3 --rows 10000000000 --steps 5 > gpurun_out/sweep/c3_10b.json 2> gpurun_out/sweep/c3_10b.log
ls gpurun_out/sweep
