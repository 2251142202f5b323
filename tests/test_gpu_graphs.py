"""CUDA-graph replay of repeated K12 plans (k_groupfused.cu run_graph): the
second call of a plan on the same user handles is captured, later calls
replay it. Replays read the columns' current contents, return fresh output
arrays, agree with a run that never uses graphs, and keep the profiled
region's timings."""
import ctypes as C
import json

import numpy as np
import pytest

from paper_2506_10092_b200 import datagen as G
from paper_2506_10092_b200 import host as H

pytestmark = pytest.mark.gpu


def _table(rng, n):
    e = G.run_ends(n, 400, rng)
    s = np.concatenate([[0], e[:-1] + 1]).astype(np.int64)
    key = H.RleColumn(rng.integers(0, 7, len(e)).astype(np.int64), s, e.astype(np.int64), n)
    pe = G.run_ends(n, 60, rng)
    ps = np.concatenate([[0], pe[:-1] + 1]).astype(np.int64)
    pred = H.RleColumn(rng.integers(0, 10, len(pe)).astype(np.int64), ps, pe.astype(np.int64), n)
    return key, pred


def _want(key, pred, vals, lim):
    """numpy: per key, SUM(v) and COUNT(*) over rows with pred < lim."""
    n = key.total_size
    k = np.repeat(key.v, key.e - key.s + 1)
    p = np.repeat(pred.v, pred.e - pred.s + 1)
    sel = p < lim
    ks = np.unique(k[sel])
    return ks, [np.array([vals[sel & (k == g)].sum() for g in ks], np.int64),
                np.array([(sel & (k == g)).sum() for g in ks], np.int64)]


def test_replay_reads_current_contents_and_returns_fresh_outputs(rq):
    rng = np.random.default_rng(5)
    n = 2_000_000
    key, pred = _table(rng, n)
    X = rq.X
    arr = rq.alloc_array(H.I32, n)
    v1 = rng.integers(-1000, 1000, n).astype(np.int32)
    keep = arr.write(0, v1)
    col = rq.make_plain(arr, H.I64)
    dk, dp = rq.upload(key), rq.upload(pred)

    def call():
        ks, vs, ng, fused = rq.agg.group_aggregate_exprs(None, [dk], [X.col(col), X.count()], ["sum", "count"],
                                                         where=[(dp, "<", 5)])
        assert fused
        return ks, vs

    outs = [call() for _ in range(3)]  # direct, captured, replayed
    wk, wv = _want(key, pred, v1.astype(np.int64), 5)
    for ks, vs in outs:
        got = rq.download_all(list(ks) + list(vs))
        np.testing.assert_array_equal(got[0], wk)
        np.testing.assert_array_equal(got[1], wv[0])
        np.testing.assert_array_equal(got[2], wv[1])
    # new contents under the same handle: the replay sees them
    v2 = rng.integers(-1000, 1000, n).astype(np.int32)
    keep2 = arr.write(0, v2)
    arr.ctx.synchronize()
    ks4, vs4 = call()
    wk2, wv2 = _want(key, pred, v2.astype(np.int64), 5)
    got4 = rq.download_all(list(ks4) + list(vs4))
    np.testing.assert_array_equal(got4[1], wv2[0])
    # the previous call's outputs are untouched by the replay
    got3 = rq.download_all(list(outs[2][0]) + list(outs[2][1]))
    np.testing.assert_array_equal(got3[1], wv[0])
    del keep, keep2


def test_replays_match_ungraphed_runs_and_keep_profile(rq):
    from paper_2506_10092_b200 import queries as Q
    t = Q.lineitem_q6(3_000_000, 11)
    d = {k: rq.upload(v) for k, v in t.items()}
    ctx = d["l_shipdate"].ctx
    L = rq._L
    buf = (C.c_char * 65536)()
    L.rq_ctx_profile_only(ctx.handle, b"xg_rows")
    L.rq_ctx_set_profiling(ctx.handle, 1)
    try:
        vals = [Q.q6_fused(rq, d)[0] for _ in range(6)]
        L.rq_ctx_profile_report(ctx.handle, 1, buf, 65536)
        rep = json.loads(buf.value.decode())
    finally:
        L.rq_ctx_set_profiling(ctx.handle, 0)
        L.rq_ctx_profile_only(ctx.handle, None)
    assert len(set(np.float64(v).tobytes() for v in vals)) == 1
    assert rep["xg_rows"]["count"] == 6 and rep["xg_rows"]["ms"] > 0
    # the same plan through fresh handles never replays a graph: same bits
    d2 = {k: rq.upload(v) for k, v in t.items()}
    assert np.float64(Q.q6_fused(rq, d2)[0]).tobytes() == np.float64(vals[0]).tobytes()
