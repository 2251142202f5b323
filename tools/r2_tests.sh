# gpu parity suite (+ optional pytest args), log into gpurun_out/
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q "$@" > gpurun_out/r2_pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2_pytest_gpu.log
tail -30 gpurun_out/r2_pytest_gpu.log
