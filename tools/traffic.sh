set -x
for q in c2 c1 c3 q6 q1 c5; do
  timeout 600 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/traffic_$q.csv python tools/ncu_query.py $q > gpurun_out/traffic_$q.log 2>&1
done
ls -la gpurun_out
