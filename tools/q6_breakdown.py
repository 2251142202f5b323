"""Per-call wall-time breakdown of the fused Q6 / C5 plans (device resident)."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_10092_b200 import queries as Q
from paper_2506_10092_b200 import runq

which = sys.argv[1] if len(sys.argv) > 1 else "q6"
ctx = runq.Context(0)
if which == "q6":
    t = {k: runq.upload(v, ctx) for k, v in Q.lineitem_q6(600_000_000, 42).items()}
else:
    h = Q.production_table(750_000_000, 5)
    t = {k: runq.upload(h[k], ctx) for k in ("r2", "r3", "r4", "pi0", "p1")}
C, M, X = runq.compute, runq.masks, runq.X
times = {}


def tm(name, f):
    ctx.synchronize()
    t0 = time.perf_counter()
    r = f()
    ctx.synchronize()
    times[name] = times.get(name, 0.0) + (time.perf_counter() - t0) * 1e3
    return r


for it in range(6):
    if it == 1:
        times.clear()
    if which == "q6":
        a = tm("cmp shipdate>=", lambda: C.compare_scalar(t["l_shipdate"], Q.Q6_LO, ">="))
        b = tm("cmp shipdate<", lambda: C.compare_scalar(t["l_shipdate"], Q.Q6_HI, "<"))
        ab = tm("and1", lambda: M.and_mask(a, b))
        c = tm("cmp disc>=", lambda: C.compare_scalar(t["l_discount"], 5, ">="))
        d = tm("cmp disc<=", lambda: C.compare_scalar(t["l_discount"], 7, "<="))
        cd = tm("and2", lambda: M.and_mask(c, d))
        e = tm("cmp qty<", lambda: C.compare_scalar(t["l_quantity"], 24, "<"))
        cde = tm("and3", lambda: M.and_mask(cd, e))
        m = tm("and4", lambda: M.and_mask(ab, cde))
        tm("exprs", lambda: runq.agg.group_aggregate_exprs(
            m, [], [X.col(t["l_extendedprice"]).arith(X.col(t["l_discount"]), "*")], ["sum"]))
    else:
        m = tm("mask", lambda: Q.c5_mask(runq, t))
        tm("exprs", lambda: runq.agg.group_aggregate_exprs(m, [t["r4"]], [X.col(t["pi0"]), X.col(t["p1"]), X.count()],
                                                           Q.C5_FNS))
for k, v in times.items():
    print(f"{k:16s} {v / 5:8.3f} ms")
print(f"{'total':16s} {sum(times.values()) / 5:8.3f} ms")
