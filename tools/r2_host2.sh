set -u
mkdir -p gpurun_out/host2
for wl in q6 c5; do
  timeout 600 python tools/q_host.py $wl 100 > gpurun_out/host2/$wl.txt 2>&1
  RQ_NO_GRAPH=1 timeout 600 python tools/q_host.py $wl 100 > gpurun_out/host2/${wl}_nograph.txt 2>&1
done
