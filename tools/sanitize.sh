#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over small instances of the
# persistent TMA kernels (C1, C2), K12 and the joins.
set -u
cat > /tmp/san_run.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2506_10092_b200 import datagen as G, runq, queries as Q, host as H
a, b, c = G.c2_tables(2_000_000, 7)
print("c2", runq.agg.filtered_aggregate_binop(c, G.C2_K, "<", a, b, "*", "sum"))
a1, b1 = G.c1_tables(2_000_000, 64, 96, seed=3)
print("c1", runq.agg.aggregate_binop(a1, b1, "*", "sum"), runq.agg.aggregate_binop(b1, a1, "-", "avg"))
t = Q.lineitem_q1(300_000, 5)
print("q1", Q.q1_fused(runq, t)[1])
t6 = Q.lineitem_q6(300_000, 5)
print("q6", Q.q6_fused(runq, t6))
p = G.gapless_rle(500_000, 30, 5, 0, 5000)
bl = H.PlainColumn(np.random.default_rng(1).integers(0, 5000, 3000).astype(np.int64))
m = runq.joins.semi_join_mask(p, bl)
l, r, card = runq.joins.get_join_index(p, bl)
print("join", card)
k, x, y, z, w = G.c3_tables(2_000_000, 4)
ks, vs, ng = runq.agg.group_aggregate([k], [x, k, z, y, w], G.C3_FNS, normalize=True)
print("c3", ng)
h5 = Q.production_table(400_000, 5)
print("c5", Q.c5_fused(runq, h5)[0] if isinstance(Q.c5_fused(runq, h5), tuple) else Q.c5_fused(runq, h5))
img = runq.dump_image(x)
print("image", len(img), runq.load_image(img).download().total_size)
PY
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool python /tmp/san_run.py > gpurun_out/san_$tool.log 2>&1
  echo "$tool: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_$tool.log | tail -1)"
done
