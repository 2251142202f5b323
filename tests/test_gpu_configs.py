"""GPU parity at config level (VERDICT r1 "What's weak" 1): the whole group
tables of C3, C4 Q1 / Q6 and C5 — keys and every aggregate column — against

  * the unmodified reference library (group_aggregate over normalize_basic'd
    columns, exactly as runner.cpp:306-336 calls it) at 2–5M rows, and
  * the streaming oracle (oracle/streaming.py, pinned against the reference in
    tests/test_oracle_streaming_cpu.py) at 100M+ rows,

for both device paths (the fused kernels and the materialising operator
chain). Integers and counts bit-exact; f64 within 1e-9 relative."""
import numpy as np
import pytest

from paper_2506_10092_b200 import datagen as G
from paper_2506_10092_b200 import queries as Q
from test_oracle_streaming_cpu import tables_equal

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def so(oracle_built):
    from oracle.streaming import StreamingOracle
    return StreamingOracle()


def dev_table(rq, ks, vs):
    h = rq.download_all(list(ks) + list(vs))
    return h[:len(ks)], h[len(ks):]


def c3_device(rq, d):
    return rq.agg.group_aggregate([d["k"]], [d["x"], d["k"], d["z"], d["y"], d["w"]], G.C3_FNS, normalize=True)


@pytest.mark.parametrize("n,seed", [(4096, 1), (3_000_000, 42), (5_000_000, 9)])
def test_c3_vs_reference_group_aggregate(rq, ref, n, seed):
    k, x, y, z, w = G.c3_tables(n, seed)
    wk, wv, wng = ref.group_aggregate([ref.normalize_basic(k)],
                                      [ref.normalize_basic(c) for c in (x, k, z, y, w)], G.C3_FNS)
    d = {"k": rq.upload(k), "x": rq.upload(x), "y": rq.upload(y), "z": rq.upload(z), "w": rq.upload(w)}
    ks, vs, ng = c3_device(rq, d)
    assert ng == wng
    tables_equal(dev_table(rq, ks, vs), wk, wv)


def test_c3_streamed_upload_vs_oracle_200m(rq, so):
    """C3 at 200M rows with Z / W streamed into HBM chunk by chunk
    (rq_arr_alloc + rq_arr_write, the 10B-row path) and folded into the
    streaming oracle chunk by chunk."""
    from oracle import streaming as S
    from paper_2506_10092_b200 import host as H
    n = 200_000_000
    k, x, y, _, _ = G.c3_run_columns(n, 42)
    fold = S.C3Fold(so, k, x, y)
    za = rq.alloc_array(H.I16, n)
    wa = rq.alloc_array(H.F64, n)
    for r0 in range(0, n, G.GEN_CHUNK):
        r1 = min(n, r0 + G.GEN_CHUNK)
        z, w = G.c3_plain_rows(n, 42, r0, r1)
        keep = (za.write(r0, z), wa.write(r0, w))
        za.ctx.synchronize()
        del keep
        fold.add_plain_chunk(r0, H.PlainColumn(z, H.I64, 0), w)
    d = {"k": rq.upload(k), "x": rq.upload(x), "y": rq.upload(y), "z": rq.make_plain(za, H.I64, 0),
         "w": rq.make_plain(wa)}
    ks, vs, ng = c3_device(rq, d)
    tables_equal(dev_table(rq, ks, vs), *fold.result())


@pytest.mark.parametrize("n", [3_000_000])
def test_q1_vs_reference_full_table(rq, ref, n):
    from oracle.refpy import RefAPI
    t = Q.lineitem_q1(n, 43)
    wk, wv, _ = Q.q1(RefAPI(ref), t)
    d = {k: rq.upload(v) for k, v in t.items()}
    (ks, vs, ng), fused = Q.q1_fused(rq, d)
    assert fused
    tables_equal(dev_table(rq, ks, vs), wk, wv)


@pytest.mark.parametrize("n", [120_000_000])
def test_q1_vs_oracle(rq, so, n):
    from oracle import streaming as S
    t = Q.lineitem_q1(n, 43)
    want = S.q1(t, Q.Q1_CUTOFF, so)
    d = {k: rq.upload(v) for k, v in t.items()}
    (ks, vs, ng), fused = Q.q1_fused(rq, d)
    assert fused
    tables_equal(dev_table(rq, ks, vs), *want)
    ks, vs, ng = Q.q1(rq, d)  # the operator chain
    tables_equal(dev_table(rq, ks, vs), *want)


@pytest.mark.parametrize("n", [600_000_000])
def test_q6_vs_oracle_sf100(rq, so, n):
    from oracle import streaming as S
    t = Q.lineitem_q6(n, 42)
    want = S.q6(t, Q.Q6_WHERE, so)
    d = {k: rq.upload(v) for k, v in t.items()}
    got, fused = Q.q6_fused(rq, d)
    assert fused
    assert abs(got - want) <= 1e-9 * max(1.0, abs(got), abs(want)), (got, want)
    got = Q.q6(rq, d)
    assert abs(got - want) <= 1e-9 * max(1.0, abs(got), abs(want)), (got, want)


@pytest.mark.parametrize("n", [2_000_000, 200_000_000])
def test_c5_vs_oracle(rq, ref, so, n):
    from oracle import streaming as S
    from oracle.refpy import RefAPI
    t = Q.production_table(n, 5, columns=["r2", "r3", "r4", "pi0", "p1"])
    want = S.c5(t, Q.C5_IN, Q.C5_LT, so)
    if n <= 5_000_000:  # the reference itself at small sizes
        wk, wv, _ = Q.c5_query(RefAPI(ref), t)
        tables_equal(want, wk, wv)
    d = {k: rq.upload(t[k]) for k in ("r2", "r3", "r4", "pi0", "p1")}
    (ks, vs, ng), fused = Q.c5_fused(rq, d)
    assert fused
    tables_equal(dev_table(rq, ks, vs), *want)
    ks, vs, ng = Q.c5_query(rq, d)
    tables_equal(dev_table(rq, ks, vs), *want)


def test_f64_group_sums_bit_identical_across_runs(rq):
    """Float group sums are reproducible: the K12 row pass writes per-chunk
    partial tables folded in a fixed order (no atomics), so two runs of the
    same query give bit-identical f64 outputs."""
    t = Q.lineitem_q1(30_000_000, 43)
    d = {k: rq.upload(v) for k, v in t.items()}
    runs = []
    for _ in range(3):
        (ks, vs, ng), fused = Q.q1_fused(rq, d)
        assert fused
        runs.append(dev_table(rq, ks, vs)[1])
    for r in runs[1:]:
        for a, b in zip(runs[0], r):
            assert np.array_equal(np.asarray(a).view(np.uint64), np.asarray(b).view(np.uint64))
    t6 = Q.lineitem_q6(60_000_000, 42)
    d6 = {k: rq.upload(v) for k, v in t6.items()}
    vals = {Q.q6_fused(rq, d6)[0] for _ in range(3)}
    assert len(vals) == 1
    k, x, y, z, w = G.c3_tables(20_000_000, 5)
    dc = {"k": rq.upload(k), "x": rq.upload(x), "y": rq.upload(y), "z": rq.upload(z), "w": rq.upload(w)}
    outs = [dev_table(rq, *c3_device(rq, dc)[:2])[1] for _ in range(3)]
    for o in outs[1:]:
        for a, b in zip(outs[0], o):
            assert np.array_equal(np.asarray(a).view(np.uint64), np.asarray(b).view(np.uint64))
