"""GPU parity: the ingest side of the path on the
device — plain_to_rle / plain_to_rle_index / plain_to_plain_index, the
encoding-selection cascade (io::choose_encoding + io::encode) and the stable
lexicographic table sort (io::sort_table) — against the golden vectors and the
unmodified reference library on the reference tests' own shapes."""
import numpy as np
import pytest

from golden_io import col, load_cases
from helpers import assert_column
from paper_2506_10092_b200 import host as H

pytestmark = pytest.mark.gpu
CASES = load_cases()


def by_fn(*fns):
    return [c for c in CASES if c["fn"] in fns]


def choice_tuple(ch):
    return list(ch.as_tuple())


@pytest.mark.parametrize("case", by_fn("plain_to_plain_index"), ids=lambda c: c["name"])
def test_plain_to_plain_index_golden(rq, case):
    i = case["inputs"]
    assert_column(rq.enc.plain_to_plain_index(col(i["a"]), i["trim"]), col(case["expected"]["col"]))


@pytest.mark.parametrize("case", by_fn("choose_encoding"), ids=lambda c: c["name"])
def test_choose_encoding_golden(rq, case):
    i = case["inputs"]
    c = col(i["a"])
    ch = rq.io.choose_encoding(c, H.Heuristic(row_threshold=i["row_threshold"]))
    assert choice_tuple(ch) == case["expected"]["choice"]
    assert_column(rq.io.encode(c, ch), col(case["expected"]["col"]))


@pytest.mark.parametrize("case", by_fn("sort_table"), ids=lambda c: c["name"])
def test_sort_table_golden(rq, case):
    i = case["inputs"]
    got = rq.io.sort_table([col(c) for c in i["cols"]], i["by"])
    for g, w in zip(got, case["expected"]["cols"]):
        assert_column(g, col(w))


def _ingest_shapes(n):
    """The reference tests' 2M-row choose_encoding shapes (test_ingest.cpp:88-124)."""
    rng = np.random.default_rng(157)
    wide = np.where(rng.random(n) < 0.01, rng.integers(1_000_000, 2_000_000_000, n),
                    rng.integers(-30_000, 30_001, n))
    half = np.concatenate([np.arange(n // 2) // 100_000, 100 + np.arange(n - n // 2) % 2])
    return {
        "small_plain": np.zeros(100, np.int64),
        "long_runs": np.zeros(n, np.int64),
        "wide_outliers": wide,
        "mixed_segments": half,
        "centered": rng.integers(5_000_000_000, 5_000_000_200, n),
        "float": rng.uniform(0, 1, n),
        "narrow_storage": rng.integers(-100, 100, n).astype(np.int8),
    }


@pytest.mark.parametrize("name", list(_ingest_shapes(8).keys()))
def test_choose_and_encode_vs_reference(rq, ref, name):
    vals = _ingest_shapes(2_000_000)[name]
    c = H.PlainColumn(vals, H.I64) if vals.dtype == np.int8 else H.PlainColumn(vals)
    got, want = rq.io.choose_encoding(c), ref.choose_encoding(c)
    assert choice_tuple(got) == choice_tuple(want)
    assert_column(rq.io.encode(c, got), ref.encode(c, want))
    expect = {"small_plain": H.SCHEME_PLAIN, "long_runs": H.SCHEME_RLE, "wide_outliers": H.SCHEME_PLAIN_INDEX,
              "mixed_segments": H.SCHEME_RLE_INDEX}
    if name in expect:
        assert got.scheme == expect[name]


@pytest.mark.parametrize("trim", [0.0, 0.05, 0.3])
def test_plain_to_plain_index_5m_vs_reference(rq, ref, trim):
    rng = np.random.default_rng(int(trim * 100) + 3)
    n = 5_000_000
    v = rng.integers(-1000, 1000, n)
    v[rng.random(n) < 0.003] = rng.integers(-(1 << 50), 1 << 50)
    c = H.PlainColumn(v)
    assert_column(rq.enc.plain_to_plain_index(c, trim), ref.plain_to_plain_index(c, trim))


def test_plain_to_plain_index_rejects_trim(rq):
    with pytest.raises(Exception):
        rq.enc.plain_to_plain_index(H.PlainColumn(np.arange(4)), 0.5)


def test_sort_table_1m_vs_reference(rq, ref):
    rng = np.random.default_rng(9)
    n = 1_000_000
    cols = [H.PlainColumn(rng.integers(0, 3, n).astype(np.int8), H.I64),
            H.PlainColumn(rng.integers(8000, 10600, n)),
            H.PlainColumn(rng.choice(np.array([0.0, -0.0, 1.25, 7.5, -3.0]), n)),
            H.PlainColumn(rng.integers(-(1 << 62), 1 << 62, n)),
            H.PlainColumn(rng.uniform(0, 1e5, n))]
    for by in ([0, 1], [2, 0], [3], [1, 3, 2]):
        got = rq.io.sort_table(cols, by)
        want = ref.sort_table(cols, by)
        for g, w in zip(got, want):
            assert_column(g, w)
