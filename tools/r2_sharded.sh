# multi-rank paths on one B200: pytest (NCCL world 1 + two processes on cuda:0), bench N=2 over the host transport
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_configs.py -x -q > gpurun_out/r2_sharded_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2_sharded_pytest.log
for wl in c2 c3 q1 c5; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --workload $wl --comm host --rows 200000000 --steps 3 --no-e2e > gpurun_out/r2_n2host_$wl.json 2> gpurun_out/r2_n2host_$wl.log
done
timeout 600 python bench.py > gpurun_out/r2_bench_c2_n1.json 2> gpurun_out/r2_bench_c2_n1.log
tail -3 gpurun_out/r2_sharded_pytest.log
