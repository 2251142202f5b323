# reference's own tests on the adapter + sharded/config parity + N=2 q1 (host transport)
set -u
mkdir -p gpurun_out
timeout 900 tests/refcheck/bin/runq_tests > gpurun_out/r2_refcheck_tests.log 2>&1; echo "exit $?" >> gpurun_out/r2_refcheck_tests.log
timeout 900 tests/refcheck/bin/runq_acceptance > gpurun_out/r2_refcheck_acceptance.log 2>&1; echo "exit $?" >> gpurun_out/r2_refcheck_acceptance.log
timeout 1500 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_configs.py -q > gpurun_out/r2_sharded_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2_sharded_pytest.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --workload q1 --comm host --rows 200000000 --steps 3 --no-e2e > gpurun_out/r2_n2host_q1.json 2> gpurun_out/r2_n2host_q1.log
tail -4 gpurun_out/r2_refcheck_tests.log; tail -8 gpurun_out/r2_refcheck_acceptance.log; tail -3 gpurun_out/r2_sharded_pytest.log
