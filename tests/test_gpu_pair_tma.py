"""GPU parity of the fused RLE×RLE aggregate (rq_aggregate_binop, K2) —
the persistent bulk-copy kernel and the merge-path kernel — against the
reference library's arith → aggregate_all chain (align.cpp:495-508,
groupby.cpp:164-172) and the C restatement oracle. Cases sweep the run-
length ratio both ways (the denser column drives; the other column's window
overflows for very dense other lists), shared run ends, every operator,
SUM / COUNT / AVG, f64 values and integer ÷0."""
import numpy as np
import pytest

from helpers import assert_scalar
from paper_2506_10092_b200 import datagen as G
from paper_2506_10092_b200 import host as H
from paper_2506_10092_b200._lib import RqError

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["tma", "merge_path"])
def pair_kernel(request, monkeypatch):
    if request.param == "merge_path":
        monkeypatch.setenv("RQ_NO_TMA", "1")
    else:
        monkeypatch.delenv("RQ_NO_TMA", raising=False)
    return request.param


def rle(n, L, seed, lo=-1000, hi=1000, flt=False):
    rng = np.random.default_rng(seed)
    e = G.run_ends(n, L, rng)
    s = np.concatenate([[0], e[:-1] + 1]).astype(np.int64)
    v = rng.uniform(lo, hi, len(e)) if flt else rng.integers(lo, hi + 1, len(e)).astype(np.int64)
    return H.RleColumn(v, s, e.astype(np.int64), n)


RATIOS = [(64, 96), (96, 64), (3, 5000), (5000, 3), (1, 1), (200, 200), (2, 1_000_000)]


@pytest.mark.parametrize("la,lb", RATIOS, ids=lambda x: str(x))
def test_pair_vs_reference(rq, ref, pair_kernel, la, lb):
    n = 3_000_000
    a, b = rle(n, la, la * 7 + 1), rle(n, lb, lb * 11 + 2)
    da, db = rq.upload(a), rq.upload(b)
    for op in ["+", "-", "*"]:
        for fn in ["sum", "count", "avg"]:
            want = ref.aggregate_all(ref.arith(a, b, op), fn)
            assert_scalar(rq.agg.aggregate_binop(da, db, op, fn), want, f"{op} {fn}")


def test_pair_shared_ends(rq, ref, pair_kernel):
    """B's runs are unions of A's runs: every B end is also an A end (ties)."""
    n = 1_000_000
    a = rle(n, 10, 5)
    keep = np.random.default_rng(6).random(len(a.e)) < 0.2
    keep[-1] = True
    eb = a.e[keep]
    sb = np.concatenate([[0], eb[:-1] + 1]).astype(np.int64)
    b = H.RleColumn(np.random.default_rng(7).integers(-9, 10, len(eb)).astype(np.int64), sb, eb, n)
    for op in ["-", "*"]:
        want = ref.aggregate_all(ref.arith(a, b, op), "sum")
        assert_scalar(rq.agg.aggregate_binop(rq.upload(a), rq.upload(b), op, "sum"), want, op)
        want = ref.aggregate_all(ref.arith(b, a, op), "sum")
        assert_scalar(rq.agg.aggregate_binop(rq.upload(b), rq.upload(a), op, "sum"), want, op + " swapped")


def test_pair_float_and_division(rq, ref, pair_kernel):
    n = 2_000_000
    a, b = rle(n, 40, 1, flt=True), rle(n, 70, 2, 1, 50)
    for op in ["+", "*", "/"]:
        want = ref.aggregate_all(ref.arith(a, b, op), "sum")
        assert_scalar(rq.agg.aggregate_binop(rq.upload(a), rq.upload(b), op, "sum"), want, op)
    ai, bi = rle(n, 40, 3, -50, 50), rle(n, 70, 4, 1, 9)
    want = ref.aggregate_all(ref.arith(ai, bi, "/"), "sum")
    assert_scalar(rq.agg.aggregate_binop(rq.upload(ai), rq.upload(bi), "/", "sum"), want, "int div")
    bz = H.RleColumn(np.zeros(len(bi.v), np.int64), bi.s, bi.e, n)
    with pytest.raises(RqError):
        rq.agg.aggregate_binop(rq.upload(ai), rq.upload(bz), "/", "sum")
    # the error flag must not leak into the next call
    assert_scalar(rq.agg.aggregate_binop(rq.upload(ai), rq.upload(bi), "/", "sum"), want, "after error")


def test_pair_large_vs_oracle(rq, orq, pair_kernel):
    a, b = G.c1_tables(200_000_000, 64, 96, seed=12)
    assert rq.agg.aggregate_binop(rq.upload(a), rq.upload(b), "+", "sum") == orq.sum_rle_binop(a, b, "+")
