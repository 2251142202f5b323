"""Small C2-shaped invocations of the fused filtered aggregate (for
compute-sanitizer / ncu runs): checks against the device operator chain."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_10092_b200 import datagen as G
from paper_2506_10092_b200 import runq

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3_000_000
a, b, c = G.c2_tables(n, 7)
da, db, dc = runq.upload(a), runq.upload(b), runq.upload(c)
for _ in range(3):
    got = runq.agg.filtered_aggregate_binop(dc, G.C2_K, "<", da, db, "*", "sum")
m = runq.compute.compare_scalar(dc, G.C2_K, "<")
want = runq.agg.aggregate_all(runq.compute.arith(runq.compute.filter(da, m), runq.compute.filter(db, m), "*"), "sum")
print("fused", got, "chain", want, "OK" if got == want else "MISMATCH")
