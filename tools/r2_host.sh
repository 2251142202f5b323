set -u
mkdir -p gpurun_out
for wl in q6 c5; do
  RQ_HOST_PROFILE=1 timeout 600 python tools/host_breakdown.py $wl 50 > gpurun_out/r2_host_$wl.txt 2>&1
done
timeout 600 python tools/q_overhead.py > gpurun_out/r2_q_overhead.txt 2>&1
cat gpurun_out/r2_host_*.txt gpurun_out/r2_q_overhead.txt
