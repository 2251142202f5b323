"""GPU parity of the persistent C2 / K2 kernels on run-end distributions far
from uniform, against the reference library's operator chains
(align.cpp:495-508 / 598-771, groupby.cpp:164-172).

Each CTA's start-up search (warp_lower_bound_pair, device_common.cuh) opens
with an interpolation round that assumes run ends spread evenly over the
rows; these inputs put most rows in a few giant runs and the rest in
one-row runs (and the reverse), leave a gap over most of the domain, and
cluster the points, so the first round brackets below, above or far from
the answer and the 32-ary rounds must recover. Integer results bit-exact."""
import zlib

import numpy as np
import pytest

from helpers import assert_scalar
from paper_2506_10092_b200 import host as H

pytestmark = pytest.mark.gpu


def skewed_ends(n, rng, giant_frac, giant_runs, head=True):
    """Run ends over [0, n): giant_frac of the rows in `giant_runs` runs (at the
    head or the tail), the remaining rows in runs of 1-3 rows."""
    g = int(n * giant_frac)
    cuts = np.sort(rng.choice(np.arange(1, g), giant_runs - 1, replace=False)) if giant_runs > 1 else []
    giant = np.concatenate([cuts, [g]]).astype(np.int64) - 1  # ends within [0, g)
    small_len = rng.integers(1, 4, (n - g) // 2 + 2)
    small = np.cumsum(small_len)
    small = small[small <= n - g] - 1
    if len(small) == 0 or small[-1] != n - g - 1:
        small = np.concatenate([small, [n - g - 1]])
    if head:
        return np.concatenate([giant, g + small]).astype(np.int64)
    return np.concatenate([small, (n - g) + giant]).astype(np.int64)


def rle_from_ends(e, n, rng, lo=-1000, hi=1000, gap=None):
    s = np.concatenate([[0], e[:-1] + 1]).astype(np.int64)
    if gap is not None:  # drop the runs inside [gap[0], gap[1])
        keep = (e < gap[0]) | (s >= gap[1])
        s, e = s[keep], e[keep]
    v = rng.integers(lo, hi + 1, len(s)).astype(np.int64)
    return H.RleColumn(v, s, e.astype(np.int64), n)


def clustered_points(n, rng, m, where):
    lo, hi = int(n * where[0]), int(n * where[1])
    p = np.unique(rng.integers(lo, hi, m)).astype(np.int64)
    return H.IndexColumn(rng.integers(-1000, 1001, len(p)).astype(np.int64), p, n)


N = 4_000_000
SHAPES = [
    # name, A ends (giant fraction, giant runs, head), C ends, points window, A gap
    ("giant_head", (0.9, 8, True), (0.95, 3, True), (0.0, 1.0), None),
    ("giant_tail", (0.9, 8, False), (0.95, 3, False), (0.0, 1.0), None),
    ("points_in_tail", (0.9, 8, True), (0.5, 2, False), (0.97, 1.0), None),
    ("points_in_head", (0.9, 8, False), (0.9, 5, True), (0.0, 0.02), None),
    ("gap_over_middle", (0.5, 4, True), (0.2, 2, True), (0.0, 1.0), (0.1, 0.9)),
]


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: s[0])
def test_c2_skewed_vs_reference(rq, ref, shape):
    name, sa, sc, pw, gap = shape
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    a = rle_from_ends(skewed_ends(N, rng, *sa), N, rng,
                      gap=None if gap is None else (int(N * gap[0]), int(N * gap[1])))
    c = rle_from_ends(skewed_ends(N, rng, *sc), N, rng, 0, 63)
    b = clustered_points(N, rng, 200_000, pw)
    da, db, dc = rq.upload(a), rq.upload(b), rq.upload(c)
    for k, cmp in ((20, "<"), (40, ">=")):
        m = ref.compare_scalar(c, k, cmp)
        want = ref.aggregate_all(ref.arith(ref.filter(a, m), ref.filter(b, m), "*"), "sum")
        assert_scalar(rq.agg.filtered_aggregate_binop(dc, k, cmp, da, db, "*", "sum"), want, f"{name} {cmp}")


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: s[0])
def test_pair_skewed_vs_reference(rq, ref, shape):
    name, sa, sc, _, gap = shape
    rng = np.random.default_rng(zlib.crc32(name.encode()) + 1)
    a = rle_from_ends(skewed_ends(N, rng, *sa), N, rng)
    b = rle_from_ends(skewed_ends(N, rng, *sc), N, rng,
                      gap=None if gap is None else (int(N * gap[0]), int(N * gap[1])))
    da, db = rq.upload(a), rq.upload(b)
    for op in ("+", "*"):
        want = ref.aggregate_all(ref.arith(a, b, op), "sum")
        assert_scalar(rq.agg.aggregate_binop(da, db, op, "sum"), want, f"{name} {op}")
        assert_scalar(rq.agg.aggregate_binop(db, da, op, "sum"), ref.aggregate_all(ref.arith(b, a, op), "sum"),
                      f"{name} {op} swapped")
