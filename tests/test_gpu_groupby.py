"""GPU parity: group-by. The fused RLE-key path (k_groupfused.cu) against the
reference group_aggregate on full-coverage inputs of every data encoding,
composite keys, the normalized (query-runner) variant for RLE+Index inputs,
and a C3-shaped table at tens of millions of rows against a numpy oracle."""
import numpy as np
import pytest

from helpers import assert_array
from paper_2506_10092_b200 import datagen as G
from paper_2506_10092_b200 import host as H
from paper_2506_10092_b200._lib import RqError

pytestmark = pytest.mark.gpu
FNS = ["sum", "count", "min", "max", "avg", "std", "var"]


def full_cover_column(rng, enc, n, flt):
    if enc == H.ENC_RLE:
        return G.random_column(rng, enc, n, flt, gaps=False, domain=30)
    if enc == H.ENC_INDEX:
        return G.random_column(rng, enc, n, flt, gaps=False, domain=30)
    if enc == H.ENC_RLE_INDEX:
        return G.random_column(rng, enc, n, flt, gaps=False, domain=30)
    if enc == H.ENC_PLAIN_INDEX:
        return G.random_column(rng, enc, n)
    return G.random_column(rng, enc, n, flt, domain=30)


@pytest.mark.parametrize("enc", [H.ENC_PLAIN, H.ENC_RLE, H.ENC_INDEX, H.ENC_PLAIN_INDEX])
@pytest.mark.parametrize("flt", [False, True])
def test_fused_groupby_vs_reference(rq, ref, enc, flt):
    if enc == H.ENC_PLAIN_INDEX and flt:
        pytest.skip("plain+index is integer-only")
    rng = np.random.default_rng(1000 + enc * 2 + flt)
    for inst in range(5):
        n = int(rng.integers(50, 6000))
        key = G.gapless_rle(n, int(rng.integers(2, 40)), int(rng.integers(1 << 30)), 0, 9)
        d = full_cover_column(rng, enc, n, flt)
        ks, vs, ng = rq.agg.group_aggregate([key], [d] * len(FNS), FNS)
        wk, wv, wng = ref.group_aggregate([key], [d] * len(FNS), FNS)
        assert ng == wng
        assert_array(ks[0], wk[0], "keys")
        for g, w, fn in zip(vs, wv, FNS):
            assert_array(g, w, fn)


def test_fused_groupby_composite_keys(rq, ref):
    rng = np.random.default_rng(77)
    for inst in range(6):
        n = int(rng.integers(100, 8000))
        k1 = G.gapless_rle(n, 300, inst, 0, 2)
        k2 = G.gapless_rle(n, 50, inst + 100, 0, 1)
        d1 = G.gapless_rle(n, 7, inst + 200)
        d2 = H.PlainColumn(rng.uniform(0, 10, n))
        fns = ["sum", "count", "avg", "sum", "max"]
        ks, vs, ng = rq.agg.group_aggregate([k1, k2], [d1, d1, d1, d2, d2], fns)
        wk, wv, wng = ref.group_aggregate([k1, k2], [d1, d1, d1, d2, d2], fns)
        assert ng == wng
        for g, w in zip(ks + vs, wk + wv):
            assert_array(g, w)


def test_rle_index_inputs(rq, ref):
    rng = np.random.default_rng(5)
    n = 5000
    key = G.gapless_rle(n, 100, 3, 0, 5)
    y = G.rle_plus_index(n, 20, 0.2, 9)
    # agg::group_aggregate rejects composites (decompose), like the reference
    with pytest.raises(RqError, match="rle\\+index"):
        rq.agg.group_aggregate([key], [y], ["sum"])
    # the runner's GroupAgg normalizes first (runner.cpp:306-336)
    for fn in FNS:
        ks, vs, ng = rq.agg.group_aggregate([key], [y], [fn], normalize=True)
        wk, wv, wng = ref.group_aggregate([ref.normalize_basic(key)], [ref.normalize_basic(y)], [fn])
        assert ng == wng
        assert_array(ks[0], wk[0])
        assert_array(vs[0], wv[0], fn)


def test_gapped_inputs_take_general_path(rq, ref):
    rng = np.random.default_rng(8)
    for inst in range(5):
        n = int(rng.integers(100, 3000))
        key = G.random_column(rng, H.ENC_RLE, n, False, True, 4)
        d = G.random_column(rng, H.ENC_RLE, n, False, True, 30)
        ks, vs, ng = rq.agg.group_aggregate([key], [d, d], ["sum", "avg"])
        wk, wv, wng = ref.group_aggregate([key], [d, d], ["sum", "avg"])
        assert ng == wng
        for g, w in zip(ks + vs, wk + wv):
            assert_array(g, w)


def numpy_group_oracle(k, cols, fns):
    """Per-row decode + np.bincount (independent of both implementations)."""
    _, kv = H.column_rows(k)
    G_ = int(kv.max()) + 1
    out = []
    for c, fn in zip(cols, fns):
        if fn == "count":
            out.append(np.bincount(kv, minlength=G_).astype(np.int64))
            continue
        _, v = H.column_rows(c)
        if fn == "sum" and v.dtype.kind != "f":
            acc = np.zeros(G_, dtype=np.int64)
            np.add.at(acc, kv, v.astype(np.int64))
            out.append(acc)
        else:
            s = np.bincount(kv, weights=v.astype(np.float64), minlength=G_)
            cnt = np.bincount(kv, minlength=G_)
            out.append(s / cnt if fn == "avg" else s)
    present = np.bincount(kv, minlength=G_) > 0
    return np.nonzero(present)[0], [o[present] for o in out]


def test_c3_shape_20m_rows(rq):
    n = 20_000_000
    k, x, y, z, w = G.c3_tables(n, seed=7)
    keys_want, vals_want = numpy_group_oracle(k, [x, k, z, y, w], G.C3_FNS)
    dk, dx, dy, dz, dw = (rq.upload(c) for c in (k, x, y, z, w))
    ks, vs, ng = rq.agg.group_aggregate([dk], [dx, dk, dz, dy, dw], G.C3_FNS, normalize=True)
    assert ng == len(keys_want)
    assert np.array_equal(ks[0].download(), keys_want)
    for g, want, fn in zip(vs, vals_want, G.C3_FNS):
        got = g.download()
        if got.dtype.kind == "f":
            assert np.allclose(got, want, rtol=1e-9, atol=1e-9), fn
        else:
            assert np.array_equal(got, want), fn


# ---- K11: sort-based grouping (float keys, wide integer key ranges) --------------------

def _check_vs_ref(rq, ref, keys, data, fns):
    ks, vs, ng = rq.agg.group_aggregate(keys, data, fns)
    wk, wv, wng = ref.group_aggregate(keys, data, fns)
    assert ng == wng
    for g, w in zip(ks, wk):
        assert_array(g, w, "keys")
    for g, w, fn in zip(vs, wv, fns):
        assert_array(g, w, fn)


@pytest.mark.parametrize("kdt", [np.float64, np.float32])
def test_float_keys_vs_reference(rq, ref, kdt):
    rng = np.random.default_rng(31)
    for inst in range(4):
        n = int(rng.integers(200, 20000))
        k = G.gapless_rle(n, int(rng.integers(2, 30)), inst, -40, 40)
        k = H.RleColumn((k.v.astype(np.float64) * 0.25).astype(kdt), k.s, k.e, n)
        k.v[k.v == 0] = -0.0 if inst % 2 else 0.0      # −0.0 and +0.0 share a group
        d = G.gapless_rle(n, 5, inst + 9)
        _check_vs_ref(rq, ref, [k], [d, d, d, d], ["sum", "count", "min", "avg"])
        pk = H.PlainColumn(rng.choice(np.array([-1.5, -0.0, 0.0, 2.25, 1e30], kdt), n))
        pd = H.PlainColumn(rng.uniform(-5, 5, n))
        _check_vs_ref(rq, ref, [pk], [pd, pd, pd], ["sum", "max", "var"])


def test_wide_int_keys_vs_reference(rq, ref):
    rng = np.random.default_rng(32)
    for inst in range(4):
        n = int(rng.integers(500, 30000))
        # keys spread over the full int64 range: no dense slot table
        vals = rng.integers(-(1 << 62), 1 << 62, 64) * 2 + 1
        k = H.PlainColumn(rng.choice(vals, n))
        d = G.gapless_rle(n, 3, inst + 50)
        _check_vs_ref(rq, ref, [k], [d, d, d], ["sum", "count", "std"])


def test_composite_wide_keys_lsd_over_columns(rq, ref):
    # two full-range int64 key columns + a float column: > 64 significant bits
    rng = np.random.default_rng(33)
    n = 12000
    a = H.PlainColumn(rng.choice(rng.integers(-(1 << 62), 1 << 62, 5), n))
    b = H.PlainColumn(rng.choice(rng.integers(-(1 << 62), 1 << 62, 7), n))
    c = H.PlainColumn(rng.choice(np.array([0.5, -2.0, 3.0]), n))
    d = H.PlainColumn(rng.integers(-100, 100, n))
    _check_vs_ref(rq, ref, [a, b, c], [d, d], ["sum", "avg"])
    _check_vs_ref(rq, ref, [c, a], [d], ["max"])


def test_sort_grouping_10m_slots_vs_numpy(rq):
    # 10M plain rows, 1M distinct wide keys: radix passes over many tiles
    rng = np.random.default_rng(34)
    n = 10_000_000
    uniq = np.unique(rng.integers(-(1 << 40), 1 << 40, 1_000_000))
    kv = uniq[rng.integers(0, len(uniq), n)]
    dv = rng.integers(-1000, 1000, n)
    ks, vs, ng = rq.agg.group_aggregate([H.PlainColumn(kv)], [H.PlainColumn(dv)] * 2, ["sum", "count"])
    want_keys, inv = np.unique(kv, return_inverse=True)
    assert ng == len(want_keys)
    assert np.array_equal(ks[0], want_keys)
    want_sum = np.zeros(ng, np.int64)
    np.add.at(want_sum, inv, dv)
    assert np.array_equal(vs[0], want_sum)
    assert np.array_equal(vs[1], np.bincount(inv, minlength=ng))
