"""GPU: the multi-GPU path inside the library (include/runq_b200.h
rq_comm_* / *_sharded). Only one B200 is available to the build, so:

  * world 1 over NCCL: a real NCCL communicator on cuda:0 — the sharded entry
    points equal the unsharded ones;
  * world 2 over the host transport: two PROCESSES on cuda:0, each running
    the device path on its row-range shard (rq_shard_host_column, cuts
    snapped to run boundaries) with the packets moved by torch.distributed
    gloo — the merged tables (C2, C3, Q1, C5, MIN/MAX, AVG recomputed from
    merged SUM / COUNT) equal the reference library's UNSHARDED results.
The merge code (pack → one all-gather → device regroup → finalize) is the
same for both transports; only the byte movement differs."""
import os
import socket

import numpy as np
import pytest

from paper_2506_10092_b200 import datagen as G
from paper_2506_10092_b200 import queries as Q
from test_oracle_streaming_cpu import tables_equal

pytestmark = pytest.mark.gpu


def dev_table(rq, ks, vs):
    h = rq.download_all(list(ks) + list(vs))
    return h[:len(ks)], h[len(ks):]


@pytest.fixture(scope="module")
def comm1(rq):
    ctx = rq.default_context()
    return rq.Comm.nccl(ctx, rq.Comm.unique_id(), 1, 0)


def test_nccl_world1_equals_unsharded(rq, comm1):
    assert comm1.info() == (1, 0, "nccl")
    a, b, c = G.c2_tables(2_000_000, seed=3)
    da, db, dc = rq.upload(a), rq.upload(b), rq.upload(c)
    want = rq.agg.filtered_aggregate_binop(dc, 20, "<", da, db, "*", "sum")
    assert rq.agg.filtered_aggregate_binop(dc, 20, "<", da, db, "*", "sum", comm=comm1) == want
    a1, b1 = G.c1_tables(1_000_000, 16, 24, seed=4)
    d1, d2 = rq.upload(a1), rq.upload(b1)
    assert rq.agg.aggregate_binop(d1, d2, "+", "sum", comm=comm1) == rq.agg.aggregate_binop(d1, d2, "+", "sum")
    for fn in ("sum", "count", "min", "max", "avg"):
        assert rq.agg.aggregate_all(d1, fn, comm=comm1) == rq.agg.aggregate_all(d1, fn), fn
    k, x, y, z, w = G.c3_tables(1_000_000, 5)
    d = [rq.upload(v) for v in (k, x, y, z, w)]
    args = ([d[0]], [d[1], d[0], d[3], d[2], d[4]], G.C3_FNS)
    got = dev_table(rq, *rq.agg.group_aggregate(*args, normalize=True, comm=comm1)[:2])
    want = dev_table(rq, *rq.agg.group_aggregate(*args, normalize=True)[:2])
    tables_equal(got, *want)


def test_nccl_world1_exprs_and_errors(rq, comm1):
    t = Q.lineitem_q1(500_000, 43)
    d = {k: rq.upload(v) for k, v in t.items()}
    X = rq.X
    price, disc, tax, qty = (d[k] for k in ("l_extendedprice", "l_discount", "l_tax", "l_quantity"))
    dp = X.col(price).arith(X.col(disc).scalar(100, "-", True), "*")
    exprs = [X.col(qty), X.col(price), dp, dp.arith(X.col(tax).scalar(100, "+"), "*"), X.col(qty),
             X.col(price), X.col(disc), X.count()]
    where = [(d["l_shipdate"], "<=", Q.Q1_CUTOFF)]
    keys = [d["l_returnflag"], d["l_linestatus"]]
    ks, vs, ng, fused = rq.agg.group_aggregate_exprs(None, keys, exprs, Q.Q1_FNS, where=where, comm=comm1)
    assert fused
    wk, wv, wng, _ = rq.agg.group_aggregate_exprs(None, keys, exprs, Q.Q1_FNS, where=where)
    tables_equal(dev_table(rq, ks, vs), *dev_table(rq, wk, wv))
    # STD / VAR do not merge exactly: rejected, not approximated
    with pytest.raises(rq.RqError, match="STD / VAR"):
        rq.agg.group_aggregate([d["l_returnflag"]], [d["l_quantity"]], ["std"], comm=comm1)


def test_merge_group_tables_disjoint_keys(rq, comm1):
    """Low-level merge: a rank's partial table passes through a world-1 merge
    unchanged (keys ascending, MIN / MAX / SUM / COUNT kept)."""
    import ctypes as C
    from paper_2506_10092_b200 import host as H
    ctx = rq.default_context()
    keys = rq.upload(np.array([3, 9, 27], np.int32))
    parts = [rq.upload(np.array([5, -2, 7], np.int64)), rq.upload(np.array([1, 1, 4], np.int64)),
             rq.upload(np.array([2.5, -1.0, 0.0])), rq.upload(np.array([8, 9, 10], np.int64))]
    fns = [H.AGG_NAMES[f] for f in ("sum", "count", "min", "max")]
    karr = (C.c_void_p * 1)(keys.handle.value)
    parr = (C.c_void_p * 4)(*[p.handle.value for p in parts])
    farr = (C.c_int32 * 4)(*fns)
    ok, op_, ng = (C.c_void_p * 1)(), (C.c_void_p * 4)(), C.c_int64()
    rq.check(rq._L.rq_merge_group_tables(ctx.handle, comm1.handle, karr, 1, parr, farr, 4, 3, C.byref(ng), ok, op_))
    assert ng.value == 3
    k = rq.DeviceArray(C.c_void_p(ok[0]), ctx).download()
    assert k.dtype == np.int32 and k.tolist() == [3, 9, 27]
    got = [rq.DeviceArray(C.c_void_p(op_[i]), ctx).download().tolist() for i in range(4)]
    assert got == [[5, -2, 7], [1, 1, 4], [2.5, -1.0, 0.0], [8, 9, 10]]


# ---------------------------------------------------------------------------
# two processes on cuda:0, host transport over gloo
# ---------------------------------------------------------------------------


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _tables():
    return {
        "c2": G.c2_tables(3_000_000, seed=11),
        "c1": G.c1_tables(2_000_000, 16, 24, seed=5),
        "c3": G.c3_tables(3_000_001, seed=3),
        "q1": Q.lineitem_q1(2_000_000, 43),
        "c5": Q.production_table(2_000_000, 5),
    }


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2506_10092_b200 import runq as rq
        from paper_2506_10092_b200 import sharding as S

        def allgather(b: bytes):
            out = [None] * world
            dist.all_gather_object(out, b)
            return out

        ctx = rq.Context(0)
        comm = rq.Comm.host(ctx, world, rank, allgather)
        T = _tables()
        res = {}
        a, b, c = T["c2"]
        sh = {k: rq.upload(v, ctx) for k, v in S.shard_table({"a": a, "b": b, "c": c}, rank, world, snap="a").items()}
        res["c2"] = rq.agg.filtered_aggregate_binop(sh["c"], 20, "<", sh["a"], sh["b"], "*", "sum", comm=comm)
        a1, b1 = T["c1"]
        sh = {k: rq.upload(v, ctx) for k, v in S.shard_table({"a": a1, "b": b1}, rank, world, snap="a").items()}
        res["c1"] = [rq.agg.aggregate_binop(sh["a"], sh["b"], "+", "sum", comm=comm),
                     rq.agg.aggregate_all(sh["a"], "avg", comm=comm), rq.agg.aggregate_all(sh["b"], "min", comm=comm),
                     rq.agg.aggregate_all(sh["a"], "max", comm=comm)]
        k, x, y, z, w = T["c3"]
        sh = {n: rq.upload(v, ctx)
              for n, v in S.shard_table({"k": k, "x": x, "y": y, "z": z, "w": w}, rank, world, snap="x").items()}
        ks, vs, _ = rq.agg.group_aggregate([sh["k"]], [sh["x"], sh["k"], sh["z"], sh["y"], sh["w"]], G.C3_FNS,
                                           normalize=True, comm=comm)
        res["c3"] = dev_table(rq, ks, vs)
        ks, vs, _ = rq.agg.group_aggregate([sh["k"]], [sh["x"], sh["z"]], ["min", "max"], comm=comm)
        res["c3mm"] = dev_table(rq, ks, vs)
        t = {n: rq.upload(v, ctx) for n, v in S.shard_table(T["q1"], rank, world, snap="l_quantity").items()}
        X = rq.X
        price, disc, tax, qty = (t[n] for n in ("l_extendedprice", "l_discount", "l_tax", "l_quantity"))
        dp = X.col(price).arith(X.col(disc).scalar(100, "-", True), "*")
        exprs = [X.col(qty), X.col(price), dp, dp.arith(X.col(tax).scalar(100, "+"), "*"), X.col(qty),
                 X.col(price), X.col(disc), X.count()]
        ks, vs, _, fused = rq.agg.group_aggregate_exprs(None, [t["l_returnflag"], t["l_linestatus"]], exprs,
                                                        Q.Q1_FNS, where=[(t["l_shipdate"], "<=", Q.Q1_CUTOFF)],
                                                        comm=comm)
        res["q1"] = dev_table(rq, ks, vs)
        cols = ("r2", "r3", "r4", "pi0", "p1")
        t = {n: rq.upload(v, ctx) for n, v in S.shard_table({c: T["c5"][c] for c in cols}, rank, world,
                                                             snap="r2").items()}
        (ks, vs, _), fused5 = Q.c5_fused(_Sharded(rq, comm), t)
        res["c5"] = dev_table(rq, ks, vs)
        res["fused"] = (fused, fused5)
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


class _Sharded:
    """runq with the communicator bound into agg.group_aggregate_exprs (so the
    plan helpers in queries.py drive the sharded entry point)."""

    def __init__(self, rq, comm):
        self.X = rq.X

        class agg:
            @staticmethod
            def group_aggregate_exprs(*a, **kw):
                kw.pop("comm", None)
                return rq.agg.group_aggregate_exprs(*a, comm=comm, **kw)

            @staticmethod
            def prepare_exprs(*a, **kw):
                kw.pop("comm", None)
                return rq.agg.prepare_exprs(*a, comm=comm, **kw)
        self.agg = agg


def test_two_ranks_one_gpu_host_transport(rq, ref):
    import torch.multiprocessing as mp
    from oracle.refpy import RefAPI
    world, port = 2, _free_port()
    mctx = mp.get_context("spawn")
    q = mctx.Queue()
    procs = [mctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=900) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    T = _tables()
    api = RefAPI(ref)
    a, b, c = T["c2"]
    m = ref.compare_scalar(c, 20, "<")
    want_c2 = ref.aggregate_all(ref.arith(ref.filter(a, m), ref.filter(b, m), "*"), "sum")
    a1, b1 = T["c1"]
    want_c1 = [ref.aggregate_all(ref.arith(a1, b1, "+"), "sum"), ref.aggregate_all(a1, "avg"),
               ref.aggregate_all(b1, "min"), ref.aggregate_all(a1, "max")]
    k, x, y, z, w = T["c3"]
    wk, wv, _ = ref.group_aggregate([ref.normalize_basic(k)], [ref.normalize_basic(v) for v in (x, k, z, y, w)],
                                    G.C3_FNS)
    mk, mv, _ = ref.group_aggregate([k], [x, z], ["min", "max"])
    q1k, q1v, _ = Q.q1(api, T["q1"])
    c5k, c5v, _ = Q.c5_query(api, T["c5"])
    for rank in range(world):  # every rank holds the same merged result
        r = results[rank]
        assert r["fused"] == (True, True)
        assert r["c2"] == want_c2
        assert r["c1"][0] == want_c1[0] and r["c1"][2:] == want_c1[2:]
        assert abs(r["c1"][1] - want_c1[1]) <= 1e-12 * max(1.0, abs(want_c1[1]))
        tables_equal(r["c3"], wk, wv)
        tables_equal(r["c3mm"], mk, mv)
        tables_equal(r["q1"], q1k, q1v)
        tables_equal(r["c5"], c5k, c5v)
