set -u
OUT=gpurun_out
mkdir -p $OUT
free -g > $OUT/r2_host_mem.txt; nproc >> $OUT/r2_host_mem.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,memory.free --format=csv >> $OUT/r2_host_mem.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/r2_pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/r2_pytest_gpu.log
timeout 600 python bench.py --workload c2 > $OUT/r2_bench_c2.json 2> $OUT/r2_bench_c2.log
