"""Pins the at-scale streaming oracle (oracle/streaming.py + runq_oracle.c
orq_seg_sum_*) against the UNMODIFIED reference library on the same seeded
C3 / Q1 / Q6 / C5 tables: the full group tables — keys,
every aggregate column — must agree bit-exactly for integers / counts and
within 1e-9 relative for f64 (runner.cpp:394-402). The 100M-row runs of the
same comparison are tools/validate_streaming_oracle.py
(profiles/r2_oracle_validation.txt)."""
import numpy as np
import pytest

from paper_2506_10092_b200 import datagen as G
from paper_2506_10092_b200 import queries as Q


def tables_equal(got, want_keys, want_vals):
    keys, vals = got
    assert len(keys) == len(want_keys)
    for g, w in zip(keys, want_keys):
        assert np.array_equal(np.asarray(g).astype(np.int64), np.asarray(w).astype(np.int64))
    assert len(vals) == len(want_vals)
    for i, (g, w) in enumerate(zip(vals, want_vals)):
        g, w = np.asarray(g), np.asarray(w)
        assert g.shape == w.shape, i
        if w.dtype.kind == "f" or g.dtype.kind == "f":
            g, w = g.astype(np.float64), w.astype(np.float64)
            nan = np.isnan(g) & np.isnan(w)
            tol = 1e-9 * np.maximum(1.0, np.maximum(np.abs(g), np.abs(w)))
            assert np.all(nan | (np.abs(g - w) <= tol)), (i, g[:4], w[:4])
        else:
            assert np.array_equal(g.astype(np.int64), w.astype(np.int64)), i


@pytest.fixture(scope="module")
def so(oracle_built):
    from oracle.streaming import StreamingOracle
    return StreamingOracle()


@pytest.mark.parametrize("n,seed", [(1_000, 3), (50_000, 5), (2_000_000, 42)])
def test_c3_vs_reference(ref, so, n, seed):
    from oracle import streaming as S
    k, x, y, z, w = G.c3_tables(n, seed)
    kk = ref.normalize_basic(k)
    ks, vs, ng = ref.group_aggregate([kk], [ref.normalize_basic(c) for c in (x, k, z, y, w)], G.C3_FNS)
    tables_equal(S.c3({"k": k, "x": x, "y": y, "z": z, "w": w}, so), ks, vs)


def test_c3_chunked_equals_whole(so):
    """Folding Z / W in row chunks (the 10B-row path) gives the same table."""
    from oracle import streaming as S
    n = 300_001
    k, x, y, z, w = G.c3_tables(n, 11)
    whole = S.c3({"k": k, "x": x, "y": y, "z": z, "w": w}, so)
    f = S.C3Fold(so, k, x, y)
    for lo in range(0, n, 77_777):
        hi = min(n, lo + 77_777)
        f.add_plain_chunk(lo, type(z)(z.values[lo:hi], z.logical, z.center), w.values[lo:hi])
    tables_equal(f.result(), *whole)


@pytest.mark.parametrize("n", [60_000, 1_000_000])
def test_q1_vs_reference(ref, so, n):
    from oracle import streaming as S
    from oracle.refpy import RefAPI
    t = Q.lineitem_q1(n, 43)
    ks, vs, ng = Q.q1(RefAPI(ref), t)
    tables_equal(S.q1(t, Q.Q1_CUTOFF, so), ks, vs)


@pytest.mark.parametrize("n", [60_000, 3_000_000])
def test_q6_vs_reference(ref, so, n):
    from oracle import streaming as S
    from oracle.refpy import RefAPI
    t = Q.lineitem_q6(n, 42)
    want = Q.q6(RefAPI(ref), t)
    got = S.q6(t, Q.Q6_WHERE, so)
    assert abs(got - want) <= 1e-9 * max(1.0, abs(got), abs(want)), (got, want)


@pytest.mark.parametrize("n", [100_000, 2_000_000])
def test_c5_vs_reference(ref, so, n):
    from oracle import streaming as S
    from oracle.refpy import RefAPI
    t = Q.production_table(n, 5)
    ks, vs, ng = Q.c5_query(RefAPI(ref), t)
    tables_equal(S.c5(t, Q.C5_IN, Q.C5_LT, so), ks, vs)


def test_where_can_empty_a_group(ref, so):
    """A key whose runs all fail the WHERE produces no group (group_on_arrays
    only yields keys that occur)."""
    from oracle import streaming as S
    from oracle.refpy import RefAPI
    t = Q.lineitem_q1(50_000, 43)
    cutoff = Q.SHIP_LO + 3  # only the earliest ship dates pass: the open (N, O) group vanishes
    api = RefAPI(ref)
    m = api.compute.compare_scalar(t["l_shipdate"], cutoff, "<=")
    f = {k: api.compute.filter(v, m) for k, v in t.items()}
    ks, vs, ng = api.agg.group_aggregate([f["l_returnflag"], f["l_linestatus"]], [f["l_quantity"]], ["sum"],
                                         normalize=True)
    so_keys, so_vals = S.q1(t, cutoff, so)
    tables_equal((so_keys, so_vals[:1]), ks, vs)


@pytest.mark.parametrize("world", [2, 3])
def test_shard_partials_merge_to_whole_table(so, world):
    """The oracle of a table cut into row-range shards (each generated alone,
    datagen part=(rank, world)) merges to the whole-table oracle — the
    multi-GPU bench gate."""
    from oracle import streaming as S
    from oracle.refpy import shard_column
    n = 1_500_007
    whole = S.c3(dict(zip("kxyzw", G.c3_tables(n, 4))), so)
    parts = [S.c3_partial(dict(zip("kxyzw", G.c3_tables(n, 4, part=(r, world), slicer=shard_column))), so)
             for r in range(world)]
    tables_equal(S.c3_finish(S.merge(parts)), *whole)
    t = Q.lineitem_q1(n, 43)
    parts = [S.q1_partial(Q.lineitem_q1(n, 43, part=(r, world), slicer=shard_column), Q.Q1_CUTOFF, so)
             for r in range(world)]
    tables_equal(S.q1_finish(S.merge(parts)), *S.q1(t, Q.Q1_CUTOFF, so))
    t = Q.lineitem_q6(n, 42)
    parts = [S.q6_partial(Q.lineitem_q6(n, 42, part=(r, world), slicer=shard_column), Q.Q6_WHERE, so)
             for r in range(world)]
    a, b = S.q6_finish(S.merge(parts)), S.q6(t, Q.Q6_WHERE, so)
    assert abs(a - b) <= 1e-9 * max(1.0, abs(a), abs(b))
    cols = ["r2", "r3", "r4", "pi0", "p1"]
    t = Q.production_table(n, 5, columns=cols)
    parts = [S.c5_partial(Q.production_table(n, 5, part=(r, world), slicer=shard_column, columns=cols), Q.C5_IN,
                          Q.C5_LT, so) for r in range(world)]
    tables_equal(S.c5_finish(S.merge(parts)), *S.c5(t, Q.C5_IN, Q.C5_LT, so))
