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
