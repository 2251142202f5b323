# A/B of altlib/<variant>/librunq_b200.so builds against the tree on one workload
# usage: bash tools/ab_variants.sh c2 v1 v2 ...
set -u
wl=$1; shift
mkdir -p gpurun_out; : > gpurun_out/ab_var.txt
for rep in 1 2 3; do
  for v in tree "$@"; do
    if [ $v = tree ]; then lib=$PWD/paper_2506_10092_b200/librunq_b200.so; else lib=$PWD/altlib/$v/librunq_b200.so; fi
    RQ_LIB_PATH=$lib timeout 600 python bench.py --workload $wl --steps 20 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); r=d['roofline']; print('$v', '$wl', round(d['ms_per_step'],5), round(r['avg_launch_ms'],5), round(r['frac'],4), d.get('oracle_match'))" >> gpurun_out/ab_var.txt
  done
done
cat gpurun_out/ab_var.txt
