"""Where a chain-path query step's time goes (wall, library profile with
host times per tagged scope, cProfile of the Python side).
python tools/chain_host.py q1 [steps]"""
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

which = sys.argv[1] if len(sys.argv) > 1 else "q1"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
rows = {"q6": 600_000_000, "q1": 600_000_000, "c5": 750_000_000}.get(which, 1_000_000_000)
w = bench.WORKLOADS[which](types.SimpleNamespace(path="chain", variant="rle", rows=rows))
from paper_2506_10092_b200 import runq  # noqa: E402

ctx = runq.Context(0)
dev = {k: runq.upload(v, ctx) for k, v in w.gen(rows, 42).items()}
for _ in range(2):
    w.query(runq, dev, "chain")
ctx.synchronize()
t0 = time.perf_counter()
for _ in range(steps):
    w.query(runq, dev, "chain")
ctx.synchronize()
print(f"{which} chain: wall {(time.perf_counter() - t0) / steps * 1e3:.2f} ms/step")
L = runq._L
buf = (C.c_char * 65536)()
L.rq_ctx_set_profiling(ctx.handle, 1)
L.rq_ctx_profile_report(ctx.handle, 1, buf, 65536)
pr = cProfile.Profile()
pr.enable()
for _ in range(steps):
    w.query(runq, dev, "chain")
ctx.synchronize()
pr.disable()
L.rq_ctx_profile_report(ctx.handle, 1, buf, 65536)
rep = json.loads(buf.value.decode())
for k, v in sorted(rep.items(), key=lambda kv: -kv[1]["ms"])[:30]:
    print(f"  {k:28s} {v['ms'] / steps:9.3f} ms  x{v['count'] / steps:.1f}")
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
