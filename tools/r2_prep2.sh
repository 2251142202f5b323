set -u
rm -rf gpurun_out/prep2; mkdir -p gpurun_out/prep2
timeout 900 python -m pytest tests/test_gpu_sharded.py -x -q --timeout 600 > gpurun_out/prep2/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/prep2/pytest.log
timeout 600 python tools/chain_host.py q1 3 > gpurun_out/prep2/chain_q1.txt 2>&1
tail -3 gpurun_out/prep2/pytest.log
