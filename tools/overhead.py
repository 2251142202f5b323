"""Per-call host overhead of the fused C2 query (tiny table: the kernel is a
few microseconds, so wall time per call ~ host path + launch + sync)."""
import ctypes as C
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_10092_b200 import datagen as G, host as H, runq  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
ctx = runq.Context(0)
a, b, c = G.c2_tables(rows, seed=1, c_variant="rle")
da, db, dc = runq.upload(a, ctx), runq.upload(b, ctx), runq.upload(c, ctx)
f = runq.agg.filtered_aggregate_binop


def bench(fn, n=2000):
    for _ in range(50):
        fn()
    ctx.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    ctx.synchronize()
    return (time.perf_counter() - t0) / n * 1e6


print("python API            %.2f us/call" % bench(lambda: f(dc, 20, "<", da, db, "*", "sum")))
L = runq._L
dt, i, fl = C.c_int32(), C.c_int64(), C.c_double()
sc = H.make_scalar(20)
cmp, op, fn = H.BINOP_NAMES["<"], H.BINOP_NAMES["*"], H.AGG_NAMES["sum"]
args = (ctx.handle, dc.handle, sc, cmp, da.handle, db.handle, op, fn, C.byref(dt), C.byref(i), C.byref(fl))
print("raw ctypes call       %.2f us/call" % bench(lambda: L.rq_filtered_aggregate_binop(*args)))
L.rq_ctx_set_profiling(ctx.handle, 1)
print("raw, profiling on     %.2f us/call" % bench(lambda: L.rq_filtered_aggregate_binop(*args)))
L.rq_ctx_set_profiling(ctx.handle, 0)
print("ctx.synchronize only  %.2f us/call" % bench(lambda: ctx.synchronize()))
