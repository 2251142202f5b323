"""Prepared fused scalar calls (agg.prepare_binop / prepare_filtered_binop:
the ctypes arguments marshalled once, the call a repeated query makes) give
the reference's results on every call, like the one-shot entry points."""
import numpy as np
import pytest

from helpers import assert_scalar
from paper_2506_10092_b200 import datagen as G

pytestmark = pytest.mark.gpu


def test_prepared_binop_vs_reference(rq, ref):
    a, b = G.c1_tables(2_000_000, 64, 96, seed=7)
    da, db = rq.upload(a), rq.upload(b)
    for op, fn in (("+", "sum"), ("*", "sum"), ("-", "count"), ("+", "avg")):
        run = rq.agg.prepare_binop(da, db, op, fn)
        want = ref.aggregate_all(ref.arith(a, b, op), fn)
        for _ in range(3):
            assert_scalar(run(), want, f"{op} {fn}")
        assert_scalar(rq.agg.aggregate_binop(da, db, op, fn), want, f"{op} {fn} one-shot")


def test_prepared_filtered_binop_vs_reference(rq, ref):
    a, b, c = G.c2_tables(3_000_000, seed=11)
    da, db, dc = rq.upload(a), rq.upload(b), rq.upload(c)
    for k, cmp, op in ((20, "<", "*"), (31.5, ">=", "+"), (7, "==", "-")):
        run = rq.agg.prepare_filtered_binop(dc, k, cmp, da, db, op, "sum")
        m = ref.compare_scalar(c, k, cmp)
        want = ref.aggregate_all(ref.arith(ref.filter(a, m), ref.filter(b, m), op), "sum")
        for _ in range(3):
            assert_scalar(run(), want, f"{cmp} {k} {op}")


def test_prepared_holds_its_handles(rq, ref):
    a, b = G.c1_tables(500_000, 16, 24, seed=3)
    run = rq.agg.prepare_binop(rq.upload(a), rq.upload(b), "+", "sum")  # no other reference to the handles
    import gc
    gc.collect()
    assert_scalar(run(), ref.aggregate_all(ref.arith(a, b, "+"), "sum"), "handles kept alive")
    assert np.isfinite(float(run()))
