"""GPU parity: the operator API (runq::compute / masks / agg) through the
C ABI against the reference library on the same inputs — structurally
(same output encoding, same arrays), the acceptance suite's differential
shape (acceptance.cpp:157-293) at reduced instance counts."""
import numpy as np
import pytest

from golden_io import arr, col, load_cases, mask, scal
from helpers import assert_array, assert_column, assert_mask, assert_scalar
from paper_2506_10092_b200 import datagen as G
from paper_2506_10092_b200 import host as H
from paper_2506_10092_b200._lib import RqError

pytestmark = pytest.mark.gpu
CASES = load_cases()
ENCS = [H.ENC_PLAIN, H.ENC_RLE, H.ENC_INDEX, H.ENC_PLAIN_INDEX, H.ENC_RLE_INDEX]
ENC_NAMES = ["plain", "rle", "index", "plain+index", "rle+index"]
MENCS = [H.MASK_PLAIN, H.MASK_RLE, H.MASK_INDEX, H.MASK_COMPOSITE]
ARITH = ["+", "-", "*"]
CMPS = ["<", "<=", "==", "!=", ">=", ">"]


def by_fn(*fns):
    return [c for c in CASES if c["fn"] in fns]


# ---- golden worked examples ------------------------------------------------------

@pytest.mark.parametrize("case", by_fn("arith", "compare", "arith_scalar", "compare_scalar", "filter",
                                       "and_mask", "aggregate_all", "group_aggregate"),
                         ids=lambda c: c["name"])
def test_golden_operator_cases(rq, case):
    i, x = case["inputs"], case["expected"]
    fn = case["fn"]
    if fn == "arith":
        assert_column(rq.compute.arith(col(i["a"]), col(i["b"]), i["op"]), col(x["col"]))
    elif fn == "compare":
        assert_mask(rq.compute.compare(col(i["a"]), col(i["b"]), i["op"]), mask(x["mask"]))
    elif fn == "arith_scalar":
        assert_column(rq.compute.arith_scalar(col(i["a"]), scal(i["k"]), i["op"]), col(x["col"]))
    elif fn == "compare_scalar":
        assert_mask(rq.compute.compare_scalar(col(i["a"]), scal(i["k"]), i["op"]), mask(x["mask"]))
    elif fn == "filter":
        assert_column(rq.compute.filter(col(i["a"]), mask(i["m"])), col(x["col"]))
    elif fn == "and_mask":
        assert_mask(rq.masks.and_mask(mask(i["a"]), mask(i["b"])), mask(x["mask"]))
    elif fn == "aggregate_all":
        assert_scalar(rq.agg.aggregate_all(col(i["a"]), i["fn"]), scal(x["value"]))
    elif fn == "group_aggregate":
        ks, vs, ng = rq.agg.group_aggregate([col(k) for k in i["keys"]], [col(d) for d in i["data"]], i["fns"])
        assert ng == x["n_groups"]
        for g, w in zip(ks, x["keys"]):
            assert_array(g, arr(w))
        for g, w in zip(vs, x["values"]):
            assert_array(g, arr(w))


@pytest.mark.parametrize("case", by_fn("sum_binop"), ids=lambda c: c["name"])
def test_golden_c1_sum(rq, case):
    i = case["inputs"]
    want = scal(case["expected"]["value"])
    a, b = col(i["a"]), col(i["b"])
    assert_scalar(rq.agg.aggregate_all(rq.compute.arith(a, b, i["op"]), "sum"), want, "chain")
    assert_scalar(rq.agg.aggregate_binop(a, b, i["op"], "sum"), want, "fused")


@pytest.mark.parametrize("case", by_fn("filtered_sum"), ids=lambda c: c["name"])
def test_golden_c2_filtered_sum(rq, case):
    i = case["inputs"]
    want = scal(case["expected"]["value"])
    a, b, c = col(i["a"]), col(i["b"]), col(i["c"])
    m = rq.compute.compare_scalar(c, i["k"], i["cmp"])
    chain = rq.agg.aggregate_all(rq.compute.arith(rq.compute.filter(a, m), rq.compute.filter(b, m), i["op"]), "sum")
    assert_scalar(chain, want, "chain")
    assert_scalar(rq.agg.filtered_aggregate_binop(c, i["k"], i["cmp"], a, b, i["op"], "sum"), want, "fused")


# ---- differential over encoding pairs ---------------------------------------------

@pytest.mark.parametrize("e1", range(5), ids=lambda e: ENC_NAMES[e])
@pytest.mark.parametrize("e2", range(5), ids=lambda e: ENC_NAMES[e])
def test_binary_ops_all_pairs(rq, ref, e1, e2):
    rng = np.random.default_rng(1000 + 10 * e1 + e2)
    for inst in range(6):
        n = int(rng.integers(1, 2000))
        a = G.random_column(rng, ENCS[e1], n, False, True, 25)
        b = G.random_column(rng, ENCS[e2], n, False, True, 25)
        for op in ARITH:
            assert_column(rq.compute.arith(a, b, op), ref.arith(a, b, op), f"arith{op} inst{inst}")
        for op in CMPS:
            assert_mask(rq.compute.compare(a, b, op), ref.compare(a, b, op), f"cmp{op} inst{inst}")


@pytest.mark.parametrize("e1", range(3), ids=lambda e: ENC_NAMES[e])
def test_float_binary_ops(rq, ref, e1):
    rng = np.random.default_rng(77 + e1)
    for e2 in range(3):
        n = int(rng.integers(10, 3000))
        a = G.random_column(rng, ENCS[e1], n, True)
        b = G.random_column(rng, ENCS[e2], n, False)
        for op in ARITH + ["/"]:
            assert_column(rq.compute.arith(a, b, op), ref.arith(a, b, op), f"arith{op}")
        for op in CMPS:
            assert_mask(rq.compute.compare(a, b, op), ref.compare(a, b, op))


def test_align_shapes_vs_reference(rq, ref):
    rng = np.random.default_rng(89)
    for e1 in range(3):
        for e2 in range(3):
            a = G.random_column(rng, ENCS[e1], 120)
            b = G.random_column(rng, ENCS[e2], 120)
            got, want = rq.compute.align(a, b), ref.align(a, b)
            assert got["kind"] == want["kind"]
            for key in ("s", "e", "p", "v1", "v2"):
                if want[key] is not None:
                    assert_array(got[key], want[key], key)


@pytest.mark.parametrize("enc", range(5), ids=lambda e: ENC_NAMES[e])
def test_scalar_ops(rq, ref, enc):
    rng = np.random.default_rng(300 + enc)
    for inst in range(5):
        n = int(rng.integers(1, 3000))
        a = G.random_column(rng, ENCS[enc], n, inst % 2 == 1)
        for k in (3, -2, 0.5):
            for op in ARITH:
                for rev in (False, True):
                    assert_column(rq.compute.arith_scalar(a, k, op, rev), ref.arith_scalar(a, k, op, rev))
            for op in CMPS:
                for rev in (False, True):
                    assert_mask(rq.compute.compare_scalar(a, k, op, rev), ref.compare_scalar(a, k, op, rev))


def test_narrow_plain_predicates(rq, ref):
    rng = np.random.default_rng(5)
    for storage, logical, center in ((np.int8, H.I64, 31), (np.int16, H.I64, -3), (np.int8, H.I8, 120),
                                     (np.int32, H.I64, None), (np.int8, H.I16, None)):
        for n in (1, 15, 16, 17, 100_003):
            v = rng.integers(np.iinfo(storage).min, np.iinfo(storage).max, n).astype(storage)
            c = H.PlainColumn(v, logical, center)
            for k in (0, 20, -100):
                for op in CMPS:
                    assert_mask(rq.compute.compare_scalar(c, k, op), ref.compare_scalar(c, k, op))
            assert_array(rq.decode_values(c), ref.decode_values(c))


def test_integer_division_by_zero_raises(rq, ref):
    a = H.RleColumn(np.array([4, 1], np.int64), [0, 5], [4, 9], 10)
    b = H.RleColumn(np.array([2, 0], np.int64), [0, 5], [4, 9], 10)
    with pytest.raises(RqError, match="division by zero"):
        rq.compute.arith(a, b, "/")
    with pytest.raises(RqError, match="division by zero"):
        rq.compute.arith_scalar(a, 0, "/")
    with pytest.raises(RqError):
        rq.compute.arith(a, H.RleColumn(np.array([1], np.int64), [0], [3], 11), "+")  # total_size mismatch
    # float division follows IEEE (align.cpp:297-301)
    f = H.RleColumn(np.array([1.0, -1.0]), [0, 5], [4, 9], 10)
    got = rq.compute.arith(f, b, "/")
    want = ref.arith(f, b, "/")
    assert_column(got, want)


@pytest.mark.parametrize("de", range(5), ids=lambda e: ENC_NAMES[e])
@pytest.mark.parametrize("me", range(4), ids=lambda e: ["plain", "rle", "index", "composite"][e])
def test_filter_all_pairs(rq, ref, de, me):
    rng = np.random.default_rng(500 + 10 * de + me)
    for inst in range(8):
        n = int(rng.integers(1, 3000))
        a = G.random_column(rng, ENCS[de], n, inst % 3 == 2)
        m = G.random_mask(rng, MENCS[me], n)
        assert_column(rq.compute.filter(a, m), ref.filter(a, m), f"inst{inst}")


def test_filter_sparse_plain_mask_and_full_cover(rq, ref):
    rng = np.random.default_rng(17)
    n = 20000
    a = G.random_column(rng, H.ENC_RLE, n)
    for dens in (0.001, 0.049, 0.051, 0.7):
        m = H.PlainMask((rng.random(n) < dens).astype(np.uint8))
        assert_column(rq.compute.filter(a, m), ref.filter(a, m))
    full = H.RleMask([0], [n - 1], n)
    for enc in ENCS:
        c = G.random_column(rng, enc, n)
        assert_column(rq.compute.filter(c, full), ref.filter(c, full))


@pytest.mark.parametrize("m1", range(4))
@pytest.mark.parametrize("m2", range(4))
def test_mask_and_all_pairs(rq, ref, m1, m2):
    rng = np.random.default_rng(40 + 4 * m1 + m2)
    for inst in range(8):
        n = int(rng.integers(1, 3000))
        a = G.random_mask(rng, MENCS[m1], n)
        b = G.random_mask(rng, MENCS[m2], n)
        assert_mask(rq.masks.and_mask(a, b), ref.and_mask(a, b), f"inst{inst}")


@pytest.mark.parametrize("m1", range(4))
@pytest.mark.parametrize("m2", range(4))
def test_mask_or_not_all_pairs(rq, ref, m1, m2):
    rng = np.random.default_rng(90 + 4 * m1 + m2)
    for inst in range(8):
        n = int(rng.integers(1, 3000))
        a = G.random_mask(rng, MENCS[m1], n)
        b = G.random_mask(rng, MENCS[m2], n)
        assert_mask(rq.masks.or_mask(a, b), ref.or_mask(a, b), f"or inst{inst}")
        assert_mask(rq.masks.not_mask(a), ref.not_mask(a), f"not inst{inst}")


@pytest.mark.parametrize("enc", range(5), ids=lambda e: ENC_NAMES[e])
def test_aggregate_all_every_fn(rq, ref, enc):
    rng = np.random.default_rng(600 + enc)
    for inst in range(6):
        n = int(rng.integers(1, 5000))
        a = G.random_column(rng, ENCS[enc], n, inst % 2 == 1, True, 30)
        for fn in ("sum", "count", "min", "max", "avg", "std", "var"):
            assert_scalar(rq.agg.aggregate_all(a, fn), ref.aggregate_all(a, fn), f"{fn} inst{inst}")


def test_aggregate_empty_column_sentinels(rq, ref):
    e = H.IndexColumn(np.array([], np.int64), [], 10)
    ef = H.IndexColumn(np.array([], np.float64), [], 10)
    for c in (e, ef):
        for fn in ("sum", "count", "min", "max", "avg", "std", "var"):
            assert_scalar(rq.agg.aggregate_all(c, fn), ref.aggregate_all(c, fn), fn)


@pytest.mark.parametrize("kenc", range(3), ids=lambda e: ENC_NAMES[e])
@pytest.mark.parametrize("denc", range(3), ids=lambda e: ENC_NAMES[e])
def test_group_aggregate_vs_reference(rq, ref, kenc, denc):
    rng = np.random.default_rng(700 + 3 * kenc + denc)
    for inst in range(6):
        n = int(rng.integers(8, 4000))
        key = G.random_column(rng, ENCS[kenc], n, False, True, 4)
        data = G.random_column(rng, ENCS[denc], n, inst % 2 == 1, True, 30)
        fns = ["sum", "count", "min", "max", "avg", "std", "var"]
        ks, vs, ng = rq.agg.group_aggregate([key], [data] * len(fns), fns)
        wk, wv, wng = ref.group_aggregate([key], [data] * len(fns), fns)
        assert ng == wng
        assert_array(ks[0], wk[0], "keys")
        for g, w, fn in zip(vs, wv, fns):
            assert_array(g, w, fn)


def test_group_aggregate_composite_keys(rq, ref):
    rng = np.random.default_rng(808)
    for inst in range(10):
        n = int(rng.integers(8, 3000))
        k1 = G.random_column(rng, [H.ENC_RLE, H.ENC_PLAIN][inst % 2], n, False, inst % 3 == 0, 3)
        k2 = G.random_column(rng, H.ENC_RLE, n, False, inst % 2 == 0, 2)
        d = G.random_column(rng, H.ENC_RLE, n, False, True, 30)
        ks, vs, ng = rq.agg.group_aggregate([k1, k2], [d, d], ["sum", "count"])
        wk, wv, wng = ref.group_aggregate([k1, k2], [d, d], ["sum", "count"])
        assert ng == wng
        for g, w in zip(ks + vs, wk + wv):
            assert_array(g, w)


def test_gapless_upload_without_starts(rq, ref):
    """A gapless RLE column may cross the C ABI without s (starts implied);
    every operator result is identical to uploading s."""
    from paper_2506_10092_b200 import datagen as G2
    a = G2.gapless_rle(50_000, 16, 1)
    b = G2.gapless_rle(50_000, 24, 2)
    a_nos = H.RleColumn(a.v, None, a.e, a.total_size)
    assert a.is_gapless() and a_nos.is_gapless()
    da = rq.upload(a_nos)
    got = da.download()
    assert np.array_equal(got.s, a.s) and np.array_equal(got.e, a.e)
    assert_column(rq.compute.arith(da, rq.upload(b), "*").download(), ref.arith(a, b, "*"))
    assert rq.agg.aggregate_binop(da, rq.upload(b), "+", "sum") == ref.aggregate_all(ref.arith(a, b, "+"), "sum")
