"""GPU parity at BASELINE-scale inputs (hundreds of millions of rows) against
the C restatement oracle's streaming versions, plus size-independent
properties: linearity of SUM, fused == operator chain."""
import numpy as np
import pytest

from helpers import assert_scalar
from paper_2506_10092_b200 import datagen as G

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("L", [(16, 24), (64, 96), (1000, 1500)])
def test_c1_sum_100m_vs_oracle(rq, orq, L):
    a, b = G.c1_tables(100_000_000, L[0], L[1], seed=42)
    da, db = rq.upload(a), rq.upload(b)
    for op in ("+", "-", "*"):
        want = orq.sum_rle_binop(a, b, op)
        assert_scalar(rq.agg.aggregate_binop(da, db, op, "sum"), want, f"fused{op}")
    # operator chain on device (materialised fragments) gives the same result
    assert_scalar(rq.agg.aggregate_all(rq.compute.arith(da, db, "+"), "sum"), orq.sum_rle_binop(a, b, "+"))
    # linearity: SUM(A+B) = SUM(A) + SUM(B) (wrapping int64)
    sa = rq.agg.aggregate_all(da, "sum")
    sb = rq.agg.aggregate_all(db, "sum")
    assert rq.agg.aggregate_binop(da, db, "+", "sum") == int(np.int64(sa) + np.int64(sb))


@pytest.mark.parametrize("variant", ["rle", "narrow"])
def test_c2_filtered_sum_200m_vs_oracle(rq, orq, variant):
    a, b, c = G.c2_tables(200_000_000, seed=42, c_variant=variant)
    want = orq.filtered_sum(c, G.C2_K, "<", a, b, "*")
    da, db, dc = rq.upload(a), rq.upload(b), rq.upload(c)
    m = rq.compute.compare_scalar(dc, G.C2_K, "<")
    chain = rq.agg.aggregate_all(rq.compute.arith(rq.compute.filter(da, m), rq.compute.filter(db, m), "*"), "sum")
    assert_scalar(chain, want, "chain")
    assert_scalar(rq.agg.filtered_aggregate_binop(dc, G.C2_K, "<", da, db, "*", "sum"), want, "fused")
