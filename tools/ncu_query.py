"""One warm query step of a bench workload inside a cudaProfilerStart/Stop range,
for `ncu --profile-from-start off` (per-kernel DRAM traffic of a whole step).

    ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        --csv --log-file gpurun_out/q1_traffic.csv python tools/ncu_query.py q1
"""
import os
import sys
import types

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "q1"
rows = {"q6": 600_000_000, "q1": 600_000_000, "c5": 750_000_000}.get(which, 1_000_000_000)
args = types.SimpleNamespace(path="fused", variant="rle", rows=rows)
w = bench.WORKLOADS[which](args)
import torch  # noqa: E402
from paper_2506_10092_b200 import runq  # noqa: E402

ctx = runq.Context(0)
dev = {k: runq.upload(v, ctx) for k, v in w.gen(rows, 42).items()}
for _ in range(2):
    w.query(runq, dev, "fused")
ctx.synchronize()
torch.cuda.cudart().cudaProfilerStart()
w.query(runq, dev, "fused")
ctx.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done", which)
