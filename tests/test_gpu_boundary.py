"""GPU: the boundary completions called through the Python mirror of the
reference API (runq.kernels / enc / compute / agg, decode_full / to_rows /
stats) against the reference library on the same inputs, or — for the
kernels helpers the reference shim does not expose — against a literal
restatement of the reference loop (kernels.cpp, column.cpp cited per test).
The reference's own unit tests cover the same functions through the C++
adapter (tests/test_gpu_refcheck.py)."""
import numpy as np
import pytest

from helpers import assert_column
from paper_2506_10092_b200 import datagen as G
from paper_2506_10092_b200 import host as H

pytestmark = pytest.mark.gpu


def test_cumsum_and_checked_sum(rq):
    x = np.random.default_rng(1).integers(-1000, 1000, 100_003)
    assert np.array_equal(rq.kernels.cumsum(x, False), np.cumsum(x))
    assert np.array_equal(rq.kernels.cumsum(x, True), np.concatenate([[0], np.cumsum(x)[:-1]]))
    assert rq.kernels.checked_sum(x) == int(x.sum())
    big = np.array([1, np.iinfo(np.int64).max - 5, 3, 7], np.int64)  # overflows at element 3 (kernels.cpp:25-26)
    with pytest.raises(rq.RqOverflowError, match="at element 3"):
        rq.kernels.cumsum(big, False)
    with pytest.raises(rq.RqOverflowError):
        rq.kernels.checked_sum(big)
    neg = np.array([np.iinfo(np.int64).min, -1], np.int64)
    with pytest.raises(rq.RqOverflowError, match="at element 1"):
        rq.kernels.cumsum(neg, True)


def test_repeat_interleave_and_range_arange(rq):
    rng = np.random.default_rng(2)
    counts = rng.integers(0, 5, 10_000)
    vals = rng.integers(-50, 50, 10_000).astype(np.int16)
    assert np.array_equal(rq.kernels.repeat_interleave(vals, counts), np.repeat(vals, counts))
    start = rng.integers(0, 1 << 40, 10_000)
    want = np.concatenate([np.arange(s, s + c) for s, c in zip(start, counts)])
    assert np.array_equal(rq.kernels.range_arange(start, counts), want)
    with pytest.raises(rq.RqError, match="negative count"):
        rq.kernels.repeat_interleave(np.array([1, 2]), np.array([1, -1]))
    with pytest.raises(rq.RqError, match="length mismatch"):
        rq.kernels.range_arange(np.array([1, 2]), np.array([1]))


def _scatter_loop(values, index, G_, op):
    """kernels.cpp:67-80 / 97-125 restated: fold in input order."""
    flt = values.dtype.kind == "f" and op != "count"
    init = {"sum": 0, "count": 0, "min": np.inf if flt else np.iinfo(np.int64).max,
            "max": -np.inf if flt else np.iinfo(np.int64).min}[op]
    out = [float(init) if flt else int(init)] * G_
    for v, g in zip(values.tolist(), index.tolist()):
        if op == "sum":
            out[g] = out[g] + (float(v) if flt else int(v))
        elif op == "count":
            out[g] += 1
        elif op == "min":
            out[g] = v if v < out[g] else out[g]
        else:
            out[g] = v if out[g] < v else out[g]
    return np.array(out, np.float64 if flt else np.int64)


@pytest.mark.parametrize("op", ["sum", "min", "max", "count"])
def test_scatter_reduce_input_order(rq, op):
    rng = np.random.default_rng(3)
    n, G_ = 20_000, 37
    idx = rng.integers(0, G_, n)
    for vals in (rng.normal(0, 1e6, n), rng.integers(-10 ** 12, 10 ** 12, n)):
        got = rq.kernels.scatter_reduce(vals, idx, G_ + 3, op)  # 3 empty groups keep the identity
        want = _scatter_loop(vals, idx, G_ + 3, op)
        if op == "sum" and want.dtype.kind == "i":
            want = want.astype(np.uint64).astype(np.int64)
        assert got.dtype == want.dtype
        assert np.array_equal(got, want), op  # bit-exact, f64 sums included
    with pytest.raises(rq.RqError, match="out of range at element 1"):
        rq.kernels.scatter_reduce(np.array([1.0, 2.0]), np.array([0, 5]), 3, "sum")


@pytest.mark.parametrize("op", ["sum", "min", "max", "count"])
def test_scatter_reduce_few_large_groups(rq, op):
    """Few groups of millions of elements take the warp-range fold: integers
    exact, f64 min / max exact, f64 sums within 1e-12 of the input-order
    loop and bit-identical run to run."""
    rng = np.random.default_rng(4)
    n, G_ = 3_000_000, 5
    idx = rng.integers(0, G_, n)
    idx[idx == 3] = 2  # one empty group keeps the identity
    for vals in (rng.normal(0, 1e6, n), rng.integers(-10 ** 12, 10 ** 12, n)):
        got = rq.kernels.scatter_reduce(vals, idx, G_, op)
        flt = vals.dtype.kind == "f" and op != "count"
        if op == "sum":
            want = np.array([vals[idx == g].sum() if flt else int(vals[idx == g].astype(object).sum())
                             for g in range(G_)], np.float64 if flt else object)
            if not flt:
                want = np.array([int(w) & ((1 << 64) - 1) for w in want], np.uint64).astype(np.int64)
        elif op == "count":
            want = np.bincount(idx, minlength=G_).astype(np.int64)
        else:
            f = np.min if op == "min" else np.max
            ident = (np.inf if op == "min" else -np.inf) if flt else \
                (np.iinfo(np.int64).max if op == "min" else np.iinfo(np.int64).min)
            want = np.array([f(vals[idx == g]) if (idx == g).any() else ident for g in range(G_)],
                            np.float64 if flt else np.int64)
        if flt and op == "sum":
            np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-3)
            again = rq.kernels.scatter_reduce(vals, idx, G_, op)
            assert got.tobytes() == again.tobytes()
        else:
            assert np.array_equal(got, want), op


def test_unique_gather_sort_adjacent(rq):
    rng = np.random.default_rng(4)
    a = rng.integers(0, 7, 5000).astype(np.int32)
    b = rng.normal(size=5000).round(1)
    keys, inv, ng = rq.kernels.unique_with_inverse([a, b])
    order = np.lexsort((b, a))
    ua = np.unique(np.stack([a.astype(np.float64), b], 1), axis=0)
    assert ng == len(ua) and np.array_equal(keys[0], ua[:, 0].astype(np.int32)) and np.array_equal(keys[1], ua[:, 1])
    assert np.array_equal(keys[0][inv], a) and np.array_equal(keys[1][inv], b)
    assert np.array_equal(rq.kernels.gather(b, order), b[order])
    with pytest.raises(rq.RqError, match="index out of range: 5000"):
        rq.kernels.gather(b, np.array([0, 5000]))
    s, perm = rq.kernels.sort_with_perm(b)
    assert np.array_equal(perm, np.argsort(b, kind="stable")) and np.array_equal(s, np.sort(b))
    x = np.array([3, 3, 1, 1, 1, 2], np.int64)
    assert rq.kernels.adjacent_ne(x).tolist() == [1, 0, 1, 0, 0, 1]


def test_enc_set_operations(rq, ref):
    rng = np.random.default_rng(5)
    s1, e1 = G.random_ranges(rng, 5000)
    s2, e2 = G.random_ranges(rng, 5000)
    s, e = rq.enc.range_union(s1, e1, s2, e2)
    cov = G._covered(5000, s1, e1) | G._covered(5000, s2, e2)
    m = ref.plain_mask_to_rle(H.PlainMask(cov.astype(np.uint8)))  # canonical runs of the union
    assert np.array_equal(s, m.s) and np.array_equal(e, m.e)
    p1, p2 = G.random_positions(rng, 4000), G.random_positions(rng, 4000)
    want = np.union1d(p1, p2)
    assert np.array_equal(rq.enc.merge_sorted_idx(p1, p2), want)
    assert np.array_equal(rq.enc.concat_sort_idx(p2[::-1].copy(), p1), want)
    cs, ce = rq.enc.complement_rle(s1, e1, 5000)
    m = ref.plain_mask_to_rle(H.PlainMask((~G._covered(5000, s1, e1)).astype(np.uint8)))
    assert np.array_equal(cs, m.s) and np.array_equal(ce, m.e)
    cs, ce = rq.enc.complement_index(p1, 4000)
    bits = np.ones(4000, bool)
    bits[p1] = False
    m = ref.plain_mask_to_rle(H.PlainMask(bits.astype(np.uint8)))
    assert np.array_equal(cs, m.s) and np.array_equal(ce, m.e)


def test_rle_expansions_and_compaction(rq):
    rng = np.random.default_rng(6)
    col = G.random_column(rng, H.ENC_RLE, 3000)
    idx = rq.enc.rle_to_index(col)
    lens = col.e - col.s + 1
    assert np.array_equal(idx.p, np.concatenate([np.arange(a, b + 1) for a, b in zip(col.s, col.e)]))
    assert np.array_equal(idx.v, np.repeat(col.v, lens))
    pl = rq.enc.rle_to_plain(col, fill=-7)
    want = np.full(3000, -7, col.v.dtype)
    for v, a, b in zip(col.v, col.s, col.e):
        want[a:b + 1] = v
    assert np.array_equal(pl.values, want)
    with pytest.raises(rq.RqResourceError, match="exceeds budget"):
        rq.enc.rle_to_plain(col, 0.0, budget=100)
    ri = G.random_column(rng, H.ENC_RLE_INDEX, 3000)
    c = rq.enc.compact_rle_index(ri)
    # restated from primitives.cpp:381-420: runs and points re-based at the running covered count
    segs = sorted([(a, b, True, i) for i, (a, b) in enumerate(zip(ri.runs.s, ri.runs.e))] +
                  [(p, p, False, i) for i, p in enumerate(ri.points.p)])
    at, rs, ps = 0, [], []
    for a, b, is_run, _ in segs:
        (rs if is_run else ps).append(at)
        at += b - a + 1
    assert np.array_equal(c.runs.s, rs) and np.array_equal(c.points.p, ps) and c.runs.total_size == at


def test_decode_full_to_rows_stats(rq, ref):
    rng = np.random.default_rng(7)
    for enc in (H.ENC_PLAIN, H.ENC_RLE, H.ENC_INDEX, H.ENC_PLAIN_INDEX, H.ENC_RLE_INDEX):
        col = G.random_column(rng, enc, 2000)
        p, v = rq.to_rows(col)
        norm = ref.normalize_basic(col)  # rows view of the reference (align.cpp:102-115 → to_rows)
        if isinstance(norm, H.PlainColumn):
            assert np.array_equal(p, np.arange(2000)) and np.array_equal(v, ref.decode_values(norm))
        elif isinstance(norm, H.IndexColumn):
            assert np.array_equal(p, norm.p) and np.array_equal(v, norm.v)
        full = G.random_column(rng, enc, 2000, gaps=False)
        assert np.array_equal(rq.decode_full(full), rq.to_rows(full)[1])
        st = rq.stats(col)
        runs = {H.ENC_RLE: lambda c: len(c.s), H.ENC_INDEX: lambda c: len(c.p),
                H.ENC_RLE_INDEX: lambda c: len(c.runs.s)}.get(enc, lambda c: 0)(col)
        assert st["n_runs"] == runs
    gapped = H.RleColumn(np.array([1, 2]), [0, 5], [2, 6], 10)
    with pytest.raises(rq.RqError, match="has gaps"):
        rq.decode_full(gapped)
    st = rq.stats(H.RleColumn(np.arange(4, dtype=np.int32), [0, 10, 20, 30], [9, 19, 29, 39], 40))
    assert st["encoded_bytes"] == 4 * 20 and st["plain_bytes"] == 160 and st["avg_run_length"] == 10.0


def test_group_and_aggregate_array(rq, ref):
    rng = np.random.default_rng(8)
    k = G.random_column(rng, H.ENC_RLE, 3000, gaps=False, domain=4)
    d = G.random_column(rng, H.ENC_PLAIN, 3000, float_vals=True)
    g = rq.agg.group([k])
    wk, wv, _ = ref.group_aggregate([k], [d, d, d, d, d], ["sum", "count", "avg", "min", "var"])
    assert g.n_groups == len(wk[0]) and np.array_equal(g.keys[0], wk[0])
    sh, vals = rq.compute.align_many([k, d])
    assert sh.kind == "dense" and np.array_equal(vals[1], d.values)
    gd = rq.agg.group_on_arrays(sh, [vals[0]], 3000)
    for fn, want in zip(["sum", "count", "avg", "min", "var"], wv):
        got = rq.agg.aggregate_array(sh, vals[1], gd, fn)
        assert got.dtype == want.dtype and np.allclose(got, want, rtol=1e-12, atol=0), fn
    assert np.array_equal(rq.agg.aggregate(d, gd, "count"), wv[1])
    ks, kv = rq.compute.decompose(k)
    assert ks.kind == "run" and np.array_equal(ks.s, k.s) and np.array_equal(kv, k.v)
    assert np.array_equal(rq.compute.shape_weights(ks), k.e - k.s + 1)
