"""CPU: pin the C restatement oracle (oracle/runq_oracle.c) against the golden
vectors (reference outputs + the reference tests' literal expectations) and
live against the unmodified reference library on seeded inputs."""
import numpy as np
import pytest

from golden_io import arr, col, i64, load_cases, mask, scal
from helpers import assert_array
from paper_2506_10092_b200 import datagen as G
from paper_2506_10092_b200 import host as H

CASES = load_cases()


def by_fn(*fns):
    return [c for c in CASES if c["fn"] in fns]


@pytest.mark.parametrize("case", by_fn("range_intersect"), ids=lambda c: c["name"])
def test_orq_range_intersect_golden(orq, case):
    i, x = case["inputs"], case["expected"]
    s, e, i1, i2 = orq.range_intersect(i["s1"], i["e1"], i["s2"], i["e2"])
    for got, key in ((s, "s"), (e, "e"), (i1, "idx1"), (i2, "idx2")):
        assert_array(got, i64(x[key]), key)
    if "literal" in case:
        assert s.tolist() == case["literal"]["s"]


@pytest.mark.parametrize("case", by_fn("idx_in_rle", "rle_contain_idx"), ids=lambda c: c["name"])
def test_orq_points_in_runs_golden(orq, case):
    i, x = case["inputs"], case["expected"]
    for fn in (orq.idx_in_rle, orq.rle_contain_idx):  # identical results (test_primitives.cpp:95-104)
        p, r, q = fn(i["p"], i["s"], i["e"])
        assert_array(p, i64(x["p_out"]), "p_out")
        assert_array(r, i64(x["run_of"]), "run_of")
        assert_array(q, i64(x["idx_of"]), "idx_of")


@pytest.mark.parametrize("case", by_fn("idx_in_idx"), ids=lambda c: c["name"])
def test_orq_idx_in_idx_golden(orq, case):
    i, x = case["inputs"], case["expected"]
    p, a, b = orq.idx_in_idx(i["p1"], i["p2"])
    assert_array(p, i64(x["p_out"]), "p_out")
    assert_array(a, i64(x["idx1"]), "idx1")
    assert_array(b, i64(x["idx2"]), "idx2")


@pytest.mark.parametrize("case", by_fn("bucketize"), ids=lambda c: c["name"])
def test_orq_bucketize_golden(orq, case):
    i, x = case["inputs"], case["expected"]
    assert_array(orq.bucketize(i["x"], i["b"], i["right"]), i64(x["out"]), "out")


@pytest.mark.parametrize("case", by_fn("plain_mask_to_rle", "plain_mask_to_index"), ids=lambda c: c["name"])
def test_orq_plain_mask_golden(orq, case):
    m = mask(case["inputs"]["m"])
    want = mask(case["expected"]["mask"])
    if case["fn"] == "plain_mask_to_rle":
        s, e = orq.plain_mask_to_rle(m.bits)
        assert_array(s, want.s, "s")
        assert_array(e, want.e, "e")
    else:
        assert_array(orq.plain_mask_to_index(m.bits), want.p, "p")


@pytest.mark.parametrize("case", by_fn("compact_rle"), ids=lambda c: c["name"])
def test_orq_compact_golden(orq, case):
    a = col(case["inputs"]["a"])
    want = col(case["expected"]["col"])
    s, e, tot = orq.compact_rle(a.s, a.e)
    assert_array(s, want.s, "s")
    assert_array(e, want.e, "e")
    assert tot == want.total_size


@pytest.mark.parametrize("case", by_fn("plain_to_rle", "plain_to_rle_index"), ids=lambda c: c["name"])
def test_orq_plain_to_rle_golden(orq, case):
    a = col(case["inputs"]["a"])
    want = col(case["expected"]["col"])
    s, e = orq.plain_to_rle_int(a.values)
    vals = orq.decode_plain_int(a.values[s], a.logical, a.center)
    if case["fn"] == "plain_to_rle":
        assert_array(s, want.s, "s")
        assert_array(e, want.e, "e")
        assert vals.tolist() == want.v.tolist()
        return
    mr = case["inputs"]["min_run"]
    long_ = (e - s + 1) >= mr
    assert_array(s[long_], want.runs.s, "s")
    assert_array(e[long_], want.runs.e, "e")
    assert vals[long_].tolist() == want.runs.v.tolist()
    pts = np.concatenate([np.arange(a, b + 1) for a, b in zip(s[~long_], e[~long_])] or [i64([])])
    assert_array(pts.astype(np.int64), want.points.p, "p")


@pytest.mark.parametrize("case", by_fn("sum_binop"), ids=lambda c: c["name"])
def test_orq_c1_sum_golden(orq, case):
    i = case["inputs"]
    assert orq.sum_rle_binop(col(i["a"]), col(i["b"]), i["op"]) == scal(case["expected"]["value"])


@pytest.mark.parametrize("case", by_fn("filtered_sum"), ids=lambda c: c["name"])
def test_orq_c2_filtered_golden(orq, case):
    i = case["inputs"]
    got = orq.filtered_sum(col(i["c"]), i["k"], i["cmp"], col(i["a"]), col(i["b"]), i["op"])
    assert got == scal(case["expected"]["value"])


def test_orq_decode_plain_matches_reference(ref, orq):
    rng = np.random.default_rng(7)
    for storage, logical, center in ((np.int8, H.I64, 100), (np.int16, H.I32, -7), (np.int8, H.I8, 120),
                                     (np.int32, H.I64, None)):
        v = rng.integers(np.iinfo(storage).min, np.iinfo(storage).max, 1000).astype(storage)
        c = H.PlainColumn(v, logical, center)
        want = ref.decode_values(c)
        assert_array(orq.decode_plain_int(v, logical, center), want.astype(np.int64), "decode", exact_dtype=False)


def test_orq_vs_reference_random(ref, orq):
    rng = np.random.default_rng(11)
    for _ in range(60):
        n = int(rng.integers(1, 3000))
        s1, e1 = G.random_ranges(rng, n)
        s2, e2 = G.random_ranges(rng, n)
        for got, want in zip(orq.range_intersect(s1, e1, s2, e2), ref.range_intersect(s1, e1, s2, e2)):
            assert_array(got, want)
        p = G.random_positions(rng, n)
        for got, want in zip(orq.rle_contain_idx(p, s1, e1), ref.rle_contain_idx(p, s1, e1)):
            assert_array(got, want)
        v = rng.integers(-5, 5, len(s1))
        so, eo = orq.rle_compare_scalar(v, s1, e1, "<", 1)
        m = ref.compare_scalar(H.RleColumn(v, s1, e1, n), 1, "<")
        assert_array(so, m.s)
        assert_array(eo, m.e)


def test_orq_streaming_c1_c2_vs_reference(ref, orq):
    for seed in range(3):
        a, b = G.c1_tables(200_000, 64, 96, seed)
        for op in ("+", "-", "*"):
            assert orq.sum_rle_binop(a, b, op) == ref.aggregate_all(ref.arith(a, b, op), "sum")
        for variant in ("rle", "narrow"):
            a2, b2, c2 = G.c2_tables(300_000, seed, variant)
            m = ref.compare_scalar(c2, G.C2_K, "<")
            want = ref.aggregate_all(ref.arith(ref.filter(a2, m), ref.filter(b2, m), "*"), "sum")
            assert orq.filtered_sum(c2, G.C2_K, "<", a2, b2, "*") == want


@pytest.mark.parametrize("case", by_fn("plain_to_plain_index", "choose_encoding", "sort_table",
                                       "plain_to_rle", "plain_to_rle_index"), ids=lambda c: c["name"])
def test_ref_ingest_golden(ref, case):
    """The reference library reproduces its own committed ingest fixtures."""
    from helpers import assert_column
    i, x = case["inputs"], case["expected"]
    fn = case["fn"]
    if fn == "sort_table":
        for g, w in zip(ref.sort_table([col(c) for c in i["cols"]], i["by"]), x["cols"]):
            assert_column(g, col(w))
    elif fn == "choose_encoding":
        ch = ref.choose_encoding(col(i["a"]), H.Heuristic(row_threshold=i["row_threshold"]))
        assert list(ch.as_tuple()) == x["choice"]
        assert_column(ref.encode(col(i["a"]), ch), col(x["col"]))
    elif fn == "plain_to_plain_index":
        assert_column(ref.plain_to_plain_index(col(i["a"]), i["trim"]), col(x["col"]))
    elif fn == "plain_to_rle":
        assert_column(ref.plain_to_rle(col(i["a"])), col(x["col"]))
    else:
        assert_column(ref.plain_to_rle_index(col(i["a"]), i["min_run"]), col(x["col"]))


def test_reference_dump_column_example(ref):
    """test_column.cpp:115-129: header fields and body length = stats bytes;
    the checker the GPU image tests compare against."""
    import json

    import numpy as np

    from paper_2506_10092_b200 import host as H
    c = H.RleColumn(v=np.array([5, 6], dtype=np.int32), s=np.array([0, 4]), e=np.array([1, 6]), total_size=8)
    img = ref.dump_column(c)
    nl = img.index(b"\n")
    hdr = json.loads(img[:nl])
    assert hdr == {"encoding": "rle", "total_size": 8, "value_type": "i32",
                   "widths": {"value": 4, "position": 8}, "runs": 2}
    assert len(img) - nl - 1 == 2 * (4 + 16)
    assert np.frombuffer(img[nl + 1:nl + 9], np.int32).tolist() == [5, 6]
