# A/B of two builds of the library (RQ_LIB_PATH) on C2 / C1, alternating
set -u
mkdir -p gpurun_out
: > gpurun_out/ab.txt
for rep in 1 2 3; do
  for lib in paper_2506_10092_b200/librunq_b200.so altlib/librunq_b200.so; do
    for wl in c2 c1; do
      RQ_LIB_PATH=$PWD/$lib timeout 600 python bench.py --workload $wl --steps 20 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); r=d['roofline']; print('$lib', '$wl', round(d['ms_per_step'],5), round(r['avg_launch_ms'],5), round(r['frac'],4))" >> gpurun_out/ab.txt
    done
  done
done
cat gpurun_out/ab.txt
