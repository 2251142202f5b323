# host-side cost split of Q6 / C5 steps (library host profile + cProfile)
set -u
mkdir -p gpurun_out/host
for wl in q6 c5; do
  timeout 600 python tools/q_host.py $wl 50 > gpurun_out/host/$wl.txt 2>&1
done
