"""Where a Q6 step's time goes: the Python plan helper (queries.q6_fused),
the bare C call with the ctypes arguments built once, and the device time
(CUDA events on the library stream). python tools/q_overhead.py"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2506_10092_b200 import host as H  # noqa: E402
from paper_2506_10092_b200 import queries as Q  # noqa: E402
from paper_2506_10092_b200 import runq  # noqa: E402

ctx = runq.Context(0)
t = {k: runq.upload(v, ctx) for k, v in Q.lineitem_q6(600_000_000, 42).items()}
stream = torch.cuda.ExternalStream(ctx.stream)


def timed(fn, n=50):
    for _ in range(5):
        fn()
    ctx.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    for _ in range(n):
        fn()
    e1.record(stream)
    e1.synchronize()
    return (time.perf_counter() - t0) / n * 1e3, e0.elapsed_time(e1) / n


print("q6_fused (python helper): wall %.3f ms, events %.3f ms" % timed(lambda: Q.q6_fused(runq, t)))
# the bare C call: arguments built once
X = runq.X
ex = (H.Expr * 1)()
ex[0].n_terms = 2
ex[0].ops[0] = H.BINOP_NAMES["*"]
for j, c in enumerate((t["l_extendedprice"], t["l_discount"])):
    ex[0].terms[j].col = c.handle.value
    ex[0].terms[j].op = -1
w = (H.Pred * len(Q.Q6_WHERE))()
for i, (c, op, k) in enumerate(Q.Q6_WHERE):
    w[i].col = t[c].handle.value
    w[i].op = H.BINOP_NAMES[op]
    w[i].k = H.make_scalar(k)
fns = (C.c_int32 * 1)(0)
ok, ov = (C.c_void_p * 1)(), (C.c_void_p * 1)()
ng, fused = C.c_int64(), C.c_int32()
out = (C.c_double * 1)()


def bare():
    runq.check(runq._L.rq_group_aggregate_where(ctx.handle, w, len(Q.Q6_WHERE), None, ok, 0, ex, fns, 1, C.byref(ng),
                                                ok, ov, C.byref(fused)))
    runq.check(runq._L.rq_arr_download(ctx.handle, C.c_void_p(ov[0]), out))
    runq._L.rq_arr_free(C.c_void_p(ov[0]))


print("bare C call + download: wall %.3f ms, events %.3f ms" % timed(bare))
