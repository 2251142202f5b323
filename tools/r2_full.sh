# full GPU suite + N=2 (host transport) bench for the group-by workloads
set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2_pytest_gpu.log
for wl in q1 q6; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --workload $wl --comm host --rows 200000000 --steps 3 --no-e2e > gpurun_out/r2_n2host_$wl.json 2> gpurun_out/r2_n2host_$wl.log
done
tail -3 gpurun_out/r2_pytest_gpu.log
