"""Host vs device split of one workload's step: wall time per step, host time
blocked in stream syncs (pseudo-tag host_sync_wait), launches and syncs per
step.  python tools/host_breakdown.py q6 [steps]"""
import ctypes as C
import json
import os
import sys
import time
import types

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "q6"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
rows = {"q6": 600_000_000, "q1": 600_000_000, "c5": 750_000_000}.get(which, 1_000_000_000)
w = bench.WORKLOADS[which](types.SimpleNamespace(path="fused", variant="rle", rows=rows))
from paper_2506_10092_b200 import runq  # noqa: E402

ctx = runq.Context(0)
dev = {k: runq.upload(v, ctx) for k, v in w.gen(rows, 42).items()}
for _ in range(3):
    w.query(runq, dev, "fused")
ctx.synchronize()
L = runq._L
buf = (C.c_char * 65536)()
L.rq_ctx_set_profiling(ctx.handle, 1)
L.rq_ctx_profile_report(ctx.handle, 1, buf, 65536)
l0 = ctx.launches
t0 = time.perf_counter()
for _ in range(steps):
    w.query(runq, dev, "fused")
ctx.synchronize()
wall = (time.perf_counter() - t0) / steps * 1e3
L.rq_ctx_profile_report(ctx.handle, 1, buf, 65536)
rep = json.loads(buf.value.decode())
sw = rep.get("host_sync_wait", {"ms": 0, "count": 0})
print(f"{which}: wall {wall:.3f} ms/step, blocked in syncs {sw['ms'] / steps:.3f} ms ({sw['count'] / steps:.1f} syncs), "
      f"host busy {wall - sw['ms'] / steps:.3f} ms, launches {(ctx.launches - l0) / steps:.1f}/step")
for k, v in sorted(rep.items(), key=lambda kv: -kv[1]["ms"]):
    if k != "host_sync_wait":
        print(f"  {k:24s} {v['ms'] / steps:8.4f} ms  x{v['count'] / steps:.1f}")
