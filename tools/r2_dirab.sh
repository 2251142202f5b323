# rank-directory block size A/B: kernel times of one warm Q6 / C5 step per RQ_DIR_SHIFT
set -u
rm -rf gpurun_out/dirab; mkdir -p gpurun_out/dirab
for x in 0 1 2 3; do
  for wl in q6 c5; do
    RQ_DIR_SHIFT=$x timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/dirab/${wl}_$x.csv python bench.py --workload $wl --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  done
done
python - <<'PY' > gpurun_out/dirab/summary.txt
import csv, glob, collections
for f in sorted(glob.glob("gpurun_out/dirab/*.csv")):
    rows = [r for r in csv.reader(open(f)) if len(r) > 10 and r[0].isdigit()]
    t = collections.defaultdict(list)
    for r in rows:
        name = r[4].split("(")[0].replace("rqb::", "")
        t[name].append(float(r[-1]))
    print(f, {k: round(sum(v[-2:]) / 2 / 1000, 2) for k, v in t.items() if k in ("k_kway_candidates", "k_xg_outliers_seg")})
PY
cat gpurun_out/dirab/summary.txt
