"""GPU parity of the fused filtered aggregate (the C2 query shape,
rq_filtered_aggregate_binop) against the reference library's operator chain
compare_scalar → filter ×2 → arith → aggregate_all (align.cpp:598-771,
groupby.cpp:164-172) on the same inputs.

The cases sweep the regimes of the persistent bulk-copy kernel: point
densities far above and far below the run density (run windows much smaller
than a tile / overflowing the staged window → global-search fallback),
gapped and gapless runs for both A and C, plain narrow C, non-int64 storage
(generic loads), float values, every comparison and arithmetic operator,
the A-index/B-RLE operand swap, partial last tiles and single-point inputs.
Integer results bit-exact; f64 within 1e-9 relative (runner.cpp:394-402)."""
import numpy as np
import pytest

from helpers import assert_scalar
from paper_2506_10092_b200 import datagen as G
from paper_2506_10092_b200 import host as H
from paper_2506_10092_b200._lib import RqError

pytestmark = pytest.mark.gpu


def rle(rng, n, L, gapped=False, lo=-1000, hi=1000, dtype=np.int64):
    e = G.run_ends(n, L, rng)
    s = np.concatenate([[0], e[:-1] + 1]).astype(np.int64)
    if gapped:  # drop every third run
        keep = rng.random(len(s)) > 0.33
        s, e = s[keep], e[keep]
    if np.issubdtype(dtype, np.floating):
        v = rng.uniform(lo, hi, len(s)).astype(dtype)
    else:
        v = rng.integers(lo, hi + 1, len(s)).astype(dtype)
    return H.RleColumn(v, s, e.astype(np.int64), n)


def index(rng, n, density, lo=-1000, hi=1000, dtype=np.int64):
    m = max(1, int(n * density))
    p = np.unique(rng.integers(0, n, m)).astype(np.int64)
    if np.issubdtype(dtype, np.floating):
        v = rng.uniform(lo, hi, len(p)).astype(dtype)
    else:
        v = rng.integers(lo, hi + 1, len(p)).astype(dtype)
    return H.IndexColumn(v, p, n)


def ref_chain(ref, c, k, cmp, a, b, op, fn):
    m = ref.compare_scalar(c, k, cmp)
    return ref.aggregate_all(ref.arith(ref.filter(a, m), ref.filter(b, m), op), fn)


CASES = [
    # name, n, A run length, B density, C run length, A gapped, C gapped
    ("c2_shape", 3_000_000, 64, 0.01, 256, False, False),
    ("dense_points", 2_000_000, 1000, 0.5, 4000, False, False),
    ("sparse_points_overflow", 20_000_000, 4, 0.0005, 16, False, False),
    ("gapped_a", 2_000_000, 64, 0.02, 256, True, False),
    ("gapped_c", 2_000_000, 64, 0.02, 256, False, True),
    ("gapped_both", 2_000_000, 32, 0.05, 64, True, True),
    ("huge_c_runs", 3_000_000, 64, 0.01, 1_000_000, False, False),
    ("one_run_each", 100_000, 1_000_000, 0.3, 1_000_000, False, False),
    ("tiny", 37, 3, 0.5, 5, False, False),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: c[0])
def test_fused_c2_vs_reference(rq, ref, case):
    name, n, la, dens, lc, ga, gc = case
    rng = np.random.default_rng(abs(hash(name)) % (2**32))
    a = rle(rng, n, la, ga)
    b = index(rng, n, dens)
    c = rle(rng, n, lc, gc, 0, 63)
    da, db, dc = rq.upload(a), rq.upload(b), rq.upload(c)
    for cmp in ["<", "<=", "==", "!=", ">=", ">"]:
        want = ref_chain(ref, c, 20, cmp, a, b, "*", "sum")
        assert_scalar(rq.agg.filtered_aggregate_binop(dc, 20, cmp, da, db, "*", "sum"), want, f"{name} {cmp}")
    for op in ["+", "-"]:
        for fn in ["sum", "count", "avg"]:
            want = ref_chain(ref, c, 31, "<", a, b, op, fn)
            got = rq.agg.filtered_aggregate_binop(dc, 31, "<", da, db, op, fn)
            assert_scalar(got, want, f"{name} {op} {fn}")


def test_fused_c2_swapped_operands(rq, ref):
    rng = np.random.default_rng(5)
    n = 1_500_000
    a, b, c = index(rng, n, 0.03), rle(rng, n, 50), rle(rng, n, 300, False, 0, 63)
    for op in ["-", "*"]:
        want = ref_chain(ref, c, 40, ">=", a, b, op, "sum")
        assert_scalar(rq.agg.filtered_aggregate_binop(rq.upload(c), 40, ">=", rq.upload(a), rq.upload(b), op, "sum"),
                      want, op)


def test_fused_c2_storage_widths_and_floats(rq, ref):
    rng = np.random.default_rng(6)
    n = 1_000_000
    for adt, bdt, cdt in [(np.int32, np.int64, np.int8), (np.int8, np.int16, np.int32),
                          (np.float64, np.int64, np.int64), (np.int64, np.float32, np.int16)]:
        a = rle(rng, n, 40, dtype=adt, lo=-100, hi=100)
        b = index(rng, n, 0.02, dtype=bdt, lo=-100, hi=100)
        c = rle(rng, n, 200, False, 0, 63, dtype=cdt)
        for op in ["+", "*"]:
            want = ref_chain(ref, c, 17, "<", a, b, op, "sum")
            got = rq.agg.filtered_aggregate_binop(rq.upload(c), 17, "<", rq.upload(a), rq.upload(b), op, "sum")
            assert_scalar(got, want, f"{adt.__name__}/{bdt.__name__}/{cdt.__name__} {op}")
    # float literal against integer codes: the comparison runs in f64
    a, b, c = rle(rng, n, 40), index(rng, n, 0.02), rle(rng, n, 200, False, 0, 63)
    want = ref_chain(ref, c, 20.5, "<", a, b, "*", "sum")
    assert_scalar(rq.agg.filtered_aggregate_binop(rq.upload(c), 20.5, "<", rq.upload(a), rq.upload(b), "*", "sum"),
                  want, "float literal")


def test_fused_c2_plain_narrow_c(rq, ref):
    rng = np.random.default_rng(7)
    n = 2_000_000
    a, b = rle(rng, n, 64), index(rng, n, 0.01)
    c = G.narrow_plain(n, 4, 64, 11)
    want = ref_chain(ref, c, 20, "<", a, b, "*", "sum")
    assert_scalar(rq.agg.filtered_aggregate_binop(rq.upload(c), 20, "<", rq.upload(a), rq.upload(b), "*", "sum"),
                  want, "narrow C")


def test_fused_c2_integer_division(rq, ref):
    rng = np.random.default_rng(8)
    n = 500_000
    a = rle(rng, n, 30, lo=-50, hi=50)
    b = index(rng, n, 0.05, lo=1, hi=9)
    c = rle(rng, n, 100, False, 0, 63)
    want = ref_chain(ref, c, 30, "<", a, b, "/", "sum")
    assert_scalar(rq.agg.filtered_aggregate_binop(rq.upload(c), 30, "<", rq.upload(a), rq.upload(b), "/", "sum"),
                  want, "div")
    bz = H.IndexColumn(np.zeros(len(b.p), np.int64), b.p, n)
    with pytest.raises(RqError):
        rq.agg.filtered_aggregate_binop(rq.upload(c), 30, "<", rq.upload(a), rq.upload(bz), "/", "sum")


def test_fused_c2_repeated_launches_stable(rq):
    """The last-CTA ticket counter must wrap back to 0 after every launch."""
    a, b, c = G.c2_tables(5_000_000, 3)
    ctx = rq.Context(0)
    da, db, dc = rq.upload(a, ctx), rq.upload(b, ctx), rq.upload(c, ctx)
    first = rq.agg.filtered_aggregate_binop(dc, G.C2_K, "<", da, db, "*", "sum")  # caches gapless flags
    l0 = ctx.launches
    assert rq.agg.filtered_aggregate_binop(dc, G.C2_K, "<", da, db, "*", "sum") == first
    assert ctx.launches - l0 == 1, "the single-launch persistent kernel must serve the C2 shape"
    for _ in range(20):
        assert rq.agg.filtered_aggregate_binop(dc, G.C2_K, "<", da, db, "*", "sum") == first
