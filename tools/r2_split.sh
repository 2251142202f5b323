# per-step host/device split and warm launch lists of the K12 queries (current HEAD)
set -u
O=gpurun_out/split
rm -rf $O; mkdir -p $O
for w in q6 c5 q1 c3 c2; do timeout 300 python tools/host_breakdown.py $w 20 > $O/host_$w.txt 2>&1; done
for wl in q6 c5; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv --log-file $O/warm_$wl.csv python bench.py --workload $wl --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
cat $O/host_*.txt
