"""GPU parity: encoding primitives (runq::enc, kernels::bucketize) through
the C ABI against the golden vectors and the reference library."""
import numpy as np
import pytest

from golden_io import col, i64, load_cases, mask
from helpers import assert_array, assert_column, assert_mask
from paper_2506_10092_b200 import datagen as G
from paper_2506_10092_b200 import host as H

pytestmark = pytest.mark.gpu
CASES = load_cases()


def by_fn(*fns):
    return [c for c in CASES if c["fn"] in fns]


@pytest.mark.parametrize("case", by_fn("range_intersect"), ids=lambda c: c["name"])
def test_range_intersect_golden(rq, case):
    i, x = case["inputs"], case["expected"]
    got = rq.enc.range_intersect(i64(i["s1"]), i64(i["e1"]), i64(i["s2"]), i64(i["e2"]))
    for g, key in zip(got, ("s", "e", "idx1", "idx2")):
        assert_array(g, i64(x[key]), key)


@pytest.mark.parametrize("case", by_fn("idx_in_rle", "rle_contain_idx"), ids=lambda c: c["name"])
def test_points_in_runs_golden(rq, case):
    i, x = case["inputs"], case["expected"]
    for fn in (rq.enc.idx_in_rle, rq.enc.rle_contain_idx):
        got = fn(i64(i["p"]), i64(i["s"]), i64(i["e"]))
        for g, key in zip(got, ("p_out", "run_of", "idx_of")):
            assert_array(g, i64(x[key]), key)


@pytest.mark.parametrize("case", by_fn("idx_in_idx"), ids=lambda c: c["name"])
def test_idx_in_idx_golden(rq, case):
    i, x = case["inputs"], case["expected"]
    got = rq.enc.idx_in_idx(i64(i["p1"]), i64(i["p2"]))
    for g, key in zip(got, ("p_out", "idx1", "idx2")):
        assert_array(g, i64(x[key]), key)


@pytest.mark.parametrize("case", by_fn("bucketize"), ids=lambda c: c["name"])
def test_bucketize_golden(rq, case):
    i, x = case["inputs"], case["expected"]
    assert_array(rq.kernels.bucketize(i64(i["x"]), i64(i["b"]), i["right"]), i64(x["out"]))


@pytest.mark.parametrize("case", by_fn("plain_mask_to_rle", "plain_mask_to_index"), ids=lambda c: c["name"])
def test_plain_mask_conversions_golden(rq, case):
    m = mask(case["inputs"]["m"])
    fn = rq.enc.plain_mask_to_rle if case["fn"] == "plain_mask_to_rle" else rq.enc.plain_mask_to_index
    assert_mask(fn(m), mask(case["expected"]["mask"]))


@pytest.mark.parametrize("case", by_fn("compact_rle"), ids=lambda c: c["name"])
def test_compact_rle_golden(rq, case):
    assert_column(rq.enc.compact_rle(col(case["inputs"]["a"])), col(case["expected"]["col"]))


@pytest.mark.parametrize("case", by_fn("plain_to_rle"), ids=lambda c: c["name"])
def test_plain_to_rle_golden(rq, case):
    assert_column(rq.enc.plain_to_rle(col(case["inputs"]["a"])), col(case["expected"]["col"]))


@pytest.mark.parametrize("case", by_fn("plain_to_rle_index"), ids=lambda c: c["name"])
def test_plain_to_rle_index_golden(rq, case):
    i = case["inputs"]
    assert_column(rq.enc.plain_to_rle_index(col(i["a"]), i["min_run"]), col(case["expected"]["col"]))


@pytest.mark.parametrize("n", [0, 1, 2, 1000, 3_000_000])
@pytest.mark.parametrize("storage", ["i8", "i16", "i32", "i64", "f32", "f64"])
def test_plain_to_rle_random_vs_reference(rq, ref, n, storage):
    rng = np.random.default_rng(n + len(storage))
    runs = np.repeat(rng.integers(-3, 4, n), rng.integers(1, 9, n))[:n]
    vals = runs.astype(np.dtype(storage.replace("i", "int").replace("f", "float")))
    if storage.startswith("f") and n > 10:
        vals[::97] = np.nan            # NaN != NaN: every NaN starts a run
        vals[5::89] = -0.0             # -0.0 == 0.0: no boundary
    if storage.startswith("i") and storage != "i64":
        c = H.PlainColumn(vals, H.I64, int(rng.integers(-1000, 1000)))
    else:
        c = H.PlainColumn(vals)
    assert_column(rq.enc.plain_to_rle(c), ref.plain_to_rle(c))
    for mr in (2, 5):
        assert_column(rq.enc.plain_to_rle_index(c, mr), ref.plain_to_rle_index(c, mr))


def test_plain_to_rle_index_rejects_min_run(rq):
    with pytest.raises(Exception):
        rq.enc.plain_to_rle_index(H.PlainColumn(np.zeros(4, np.int64)), 1)


@pytest.mark.parametrize("n", [0, 1, 7, 300, 5000, 200_000])
def test_range_intersect_random_vs_reference(rq, ref, n):
    rng = np.random.default_rng(n + 1)
    for density in (0.2, 0.5, 1.0):
        s1, e1 = G.random_ranges(rng, n, density) if n else (i64([]), i64([]))
        s2, e2 = G.random_ranges(rng, n, density) if n else (i64([]), i64([]))
        got = rq.enc.range_intersect(s1, e1, s2, e2)
        want = ref.range_intersect(s1, e1, s2, e2)
        for g, w, key in zip(got, want, ("s", "e", "idx1", "idx2")):
            assert_array(g, w, key)


def test_range_intersect_many_tiles_vs_oracle(rq, orq):
    # millions of runs: exercises the partition kernel + decoupled look-back
    # across thousands of tiles; checked against the C restatement.
    a = G.gapless_rle(20_000_000, 16, 1)
    rng = np.random.default_rng(5)
    s2, e2 = G.random_ranges(rng, 20_000_000, 0.5)
    got = rq.enc.range_intersect(a.s, a.e, s2, e2)
    want = orq.range_intersect(a.s, a.e, s2, e2)
    for g, w, key in zip(got, want, ("s", "e", "idx1", "idx2")):
        assert_array(g, w, key)


@pytest.mark.parametrize("n,dens", [(100, 0.2), (5000, 0.01), (5000, 0.9), (1_000_000, 0.3), (1_000_000, 0.0005)])
def test_points_random_vs_reference(rq, ref, n, dens):
    rng = np.random.default_rng(int(n * 7 + dens * 1000))
    s, e = G.random_ranges(rng, n, 0.5)
    p = G.random_positions(rng, n, dens)
    q = G.random_positions(rng, n, 0.3)
    for got, want in zip(rq.enc.idx_in_rle(p, s, e), ref.idx_in_rle(p, s, e)):
        assert_array(got, want)
    for got, want in zip(rq.enc.idx_in_idx(p, q), ref.idx_in_idx(p, q)):
        assert_array(got, want)
    for got, want in zip(rq.enc.idx_in_idx(q, p), ref.idx_in_idx(q, p)):
        assert_array(got, want)


def test_bucketize_random_vs_reference(rq, ref):
    rng = np.random.default_rng(9)
    b = np.sort(rng.integers(-1000, 1000, 5000))
    x = rng.integers(-1100, 1100, 100_000)
    for right in (False, True):
        assert_array(rq.kernels.bucketize(x, b, right), ref.bucketize(x, b, right))


@pytest.mark.parametrize("n", [1, 33, 4096, 1_000_003])
def test_plain_mask_conversions_random(rq, ref, n):
    rng = np.random.default_rng(n)
    for dens in (0.01, 0.5, 0.99):
        m = H.PlainMask((rng.random(n) < dens).astype(np.uint8))
        assert_mask(rq.enc.plain_mask_to_rle(m), ref.plain_mask_to_rle(m))
        assert_mask(rq.enc.plain_mask_to_index(m), ref.plain_mask_to_index(m))
