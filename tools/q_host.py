"""Host-side cost of one Q6 / C5 step: wall per step of the bench's query
(Python helper + download), the same with the library's host profile
(RQ_HOST_PROFILE=1: host wall time per tagged scope), and a cProfile of the
Python side.  python tools/q_host.py q6|c5 [steps]"""
import cProfile
import ctypes as C
import json
import os
import pstats
import sys
import time
import types

os.environ.setdefault("RQ_HOST_PROFILE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "q6"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
rows = {"q6": 600_000_000, "q1": 600_000_000, "c5": 750_000_000}.get(which, 1_000_000_000)
w = bench.WORKLOADS[which](types.SimpleNamespace(path="fused", variant="rle", rows=rows))
from paper_2506_10092_b200 import runq  # noqa: E402

ctx = runq.Context(0)
dev = {k: runq.upload(v, ctx) for k, v in w.gen(rows, 42).items()}
for _ in range(5):
    w.query(runq, dev, "fused")
ctx.synchronize()


def wall(n):
    t0 = time.perf_counter()
    for _ in range(n):
        w.query(runq, dev, "fused")
    ctx.synchronize()
    return (time.perf_counter() - t0) / n * 1e3


print(f"{which}: wall {wall(steps):.4f} ms/step (no profiling)")
L = runq._L
buf = (C.c_char * 65536)()
L.rq_ctx_set_profiling(ctx.handle, 1)
L.rq_ctx_profile_report(ctx.handle, 1, buf, 65536)
l0 = ctx.launches
wp = wall(steps)
L.rq_ctx_profile_report(ctx.handle, 1, buf, 65536)
rep = json.loads(buf.value.decode())
print(f"{which}: wall {wp:.4f} ms/step under the library profile, launches {(ctx.launches - l0) / steps:.1f}/step")
for k, v in sorted(rep.items(), key=lambda kv: -kv[1]["ms"]):
    print(f"  {k:24s} {v['ms'] / steps:8.4f} ms  x{v['count'] / steps:.1f}")
L.rq_ctx_set_profiling(ctx.handle, 0)
pr = cProfile.Profile()
pr.enable()
wall(steps)
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(18)
