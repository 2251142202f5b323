# A/B of an environment knob on one workload: bash tools/ab_env.sh q1 "RQ_JIT_PF_MIN=256" "RQ_JIT_PF_MIN=2048"
set -u
wl=$1; shift
mkdir -p gpurun_out
: > gpurun_out/ab_env.txt
for rep in 1 2 3; do
  for envs in "$@"; do
    env $envs timeout 600 python bench.py --workload $wl --steps 10 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); r=d['roofline']; print('$envs', '$wl', round(d['ms_per_step'],5), round(r['avg_launch_ms'],5), round(r['frac'],4))" >> gpurun_out/ab_env.txt
  done
done
cat gpurun_out/ab_env.txt
