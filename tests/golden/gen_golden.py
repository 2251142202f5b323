"""Generates tests/golden/fixtures.json — TEST INFRASTRUCTURE.

Every expected output below comes from running the UNMODIFIED reference
library (oracle/_ref/librunq_ref.so, compiled from
/root/reference/proj/core/src) on the listed inputs. Cases are
  * the reference tests' own worked examples (file:line cited per case;
    where the test states literal expectations they are recorded too and
    cross-checked here), and
  * seeded random instances of the hot-path primitives and operator chains.
Run:  python tests/golden/gen_golden.py   (needs oracle/_ref built)
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import refpy  # noqa: E402
from paper_2506_10092_b200 import datagen as G  # noqa: E402
from paper_2506_10092_b200 import host as H  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "fixtures.json")


def enc_col(c):
    if isinstance(c, H.PlainColumn):
        return {"enc": "plain", "values": c.values.tolist(), "dtype": H.dtype_code(c.values),
                "logical": c.logical, "center": c.center}
    if isinstance(c, H.RleColumn):
        return {"enc": "rle", "v": c.v.tolist(), "dtype": H.dtype_code(c.v), "s": c.s.tolist(),
                "e": c.e.tolist(), "total_size": c.total_size}
    if isinstance(c, H.IndexColumn):
        return {"enc": "index", "v": c.v.tolist(), "dtype": H.dtype_code(c.v), "p": c.p.tolist(),
                "total_size": c.total_size}
    if isinstance(c, H.PlainPlusIndexColumn):
        return {"enc": "plain+index", "base": enc_col(c.base), "outliers": enc_col(c.outliers)}
    return {"enc": "rle+index", "runs": enc_col(c.runs), "points": enc_col(c.points)}


def enc_mask(m):
    if isinstance(m, H.PlainMask):
        return {"enc": "plain", "bits": m.bits.tolist()}
    if isinstance(m, H.RleMask):
        return {"enc": "rle", "s": m.s.tolist(), "e": m.e.tolist(), "total_size": m.total_size}
    if isinstance(m, H.IndexMask):
        return {"enc": "index", "p": m.p.tolist(), "total_size": m.total_size}
    return {"enc": "composite", "runs": enc_mask(m.runs), "points": enc_mask(m.points)}


def arr(a):
    a = np.asarray(a)
    return {"dtype": H.dtype_code(a), "data": a.tolist()}


def scal(x):
    return {"f64": x} if isinstance(x, float) else {"i64": x}


def main():
    ref = refpy.Ref()
    cases = []

    def add(name, fn, inputs, expected, source, literal=None):
        case = {"name": name, "fn": fn, "inputs": inputs, "expected": expected, "source": source}
        if literal is not None:
            case["literal"] = literal
        cases.append(case)

    # --- worked examples -------------------------------------------------------
    r = ref.range_intersect([2], [7], [1, 4, 6], [3, 5, 8])
    lit = {"s": [2, 4, 6], "e": [3, 5, 7], "idx1": [0, 0, 0], "idx2": [0, 1, 2]}
    assert [x.tolist() for x in r] == [lit["s"], lit["e"], lit["idx1"], lit["idx2"]]
    add("range_intersect_paper", "range_intersect",
        {"s1": [2], "e1": [7], "s2": [1, 4, 6], "e2": [3, 5, 8]},
        {"s": r[0].tolist(), "e": r[1].tolist(), "idx1": r[2].tolist(), "idx2": r[3].tolist()},
        "proj/tests/test_primitives.cpp:9-15; acceptance.cpp:51-54", lit)
    r = ref.range_intersect([1, 4, 6], [3, 5, 8], [2], [7])
    assert r[2].tolist() == [0, 1, 2] and r[3].tolist() == [0, 0, 0]
    add("range_intersect_swapped", "range_intersect",
        {"s1": [1, 4, 6], "e1": [3, 5, 8], "s2": [2], "e2": [7]},
        {"s": r[0].tolist(), "e": r[1].tolist(), "idx1": r[2].tolist(), "idx2": r[3].tolist()},
        "proj/tests/test_primitives.cpp:30-38")
    r = ref.range_intersect([0, 5, 9], [2, 7, 9], [0, 5, 9], [2, 7, 9])
    add("range_intersect_self", "range_intersect",
        {"s1": [0, 5, 9], "e1": [2, 7, 9], "s2": [0, 5, 9], "e2": [2, 7, 9]},
        {"s": r[0].tolist(), "e": r[1].tolist(), "idx1": r[2].tolist(), "idx2": r[3].tolist()},
        "proj/tests/test_primitives.cpp:17-24")
    r = ref.range_intersect([0], [1], [5], [9])
    add("range_intersect_disjoint", "range_intersect",
        {"s1": [0], "e1": [1], "s2": [5], "e2": [9]},
        {"s": [], "e": [], "idx1": [], "idx2": []}, "proj/tests/test_primitives.cpp:26-28")
    assert len(r[0]) == 0

    for fname in ("idx_in_rle", "rle_contain_idx"):
        r = getattr(ref, fname)([2, 4, 7], [0, 6], [2, 7])
        assert r[0].tolist() == [2, 7] and r[1].tolist() == [0, 1]
        add(f"{fname}_paper", fname, {"p": [2, 4, 7], "s": [0, 6], "e": [2, 7]},
            {"p_out": r[0].tolist(), "run_of": r[1].tolist(), "idx_of": r[2].tolist()},
            "proj/tests/test_primitives.cpp:76-92; acceptance.cpp:55-60",
            {"p_out": [2, 7], "run_of": [0, 1]})
    r = ref.idx_in_idx([1, 3, 5], [3, 5, 7])
    assert r[0].tolist() == [3, 5]
    add("idx_in_idx_paper", "idx_in_idx", {"p1": [1, 3, 5], "p2": [3, 5, 7]},
        {"p_out": r[0].tolist(), "idx1": r[1].tolist(), "idx2": r[2].tolist()},
        "proj/tests/test_primitives.cpp:107-112", {"p_out": [3, 5]})

    for x, b, right, lit_out in (([3], [1, 3, 5], False, None), ([3], [1, 3, 5], True, None),
                                 ([0, 9, 4], [1, 3, 5], True, None)):
        out = ref.bucketize(x, b, right)
        add(f"bucketize_{len(cases)}", "bucketize", {"x": x, "b": b, "right": right},
            {"out": out.tolist()}, "proj/tests/test_kernels.cpp:34-38")

    a = H.RleColumn(np.array([4, 1, 3], np.int64), [0, 10, 20], [9, 19, 39], 40)
    b = H.RleColumn(np.array([6, 8], np.int64), [0, 15], [14, 39], 40)
    s = ref.arith(a, b, "+")
    assert s.s.tolist() == [0, 10, 15, 20] and s.v.tolist() == [10, 7, 9, 11]
    add("arith_add_paper", "arith", {"a": enc_col(a), "b": enc_col(b), "op": "+"},
        {"col": enc_col(s)}, "proj/tests/test_align.cpp:69-77; acceptance.cpp:75-84",
        {"s": [0, 10, 15, 20], "e": [9, 14, 19, 39], "v": [10, 7, 9, 11]})
    m = ref.compare(a, b, "<")
    add("compare_lt_paper", "compare", {"a": enc_col(a), "b": enc_col(b), "op": "<"},
        {"mask": enc_mask(m)}, "proj/tests/test_align.cpp:86-91")
    s = ref.arith_scalar(a, 2, "*")
    assert s.v.tolist() == [8, 2, 6]
    add("arith_scalar_mul_paper", "arith_scalar", {"a": enc_col(a), "k": scal(2), "op": "*"},
        {"col": enc_col(s)}, "proj/tests/test_align.cpp:143-152", {"v": [8, 2, 6]})
    s = ref.aggregate_all(s, "sum")
    add("sum_after_scale", "aggregate_all", {"a": enc_col(ref.arith_scalar(a, 2, "*")), "fn": "sum"},
        {"value": scal(s)}, "groupby.cpp:164-172")

    pi = H.PlainPlusIndexColumn(H.PlainColumn(np.array([1, 2, 0, 0, 3], np.int8), H.I64),
                                H.IndexColumn(np.array([10_000_000_000, 10_000_000_000], np.int64), [2, 3], 5))
    m = ref.compare_scalar(pi, 10_000_000_000, "==")
    add("compare_scalar_plain_index", "compare_scalar",
        {"a": enc_col(pi), "k": scal(10_000_000_000), "op": "=="}, {"mask": enc_mask(m)},
        "proj/tests/test_align.cpp:167-174")

    plain = H.PlainColumn(np.array([10, 20, 30], np.int64))
    f = ref.filter(plain, H.PlainMask(np.array([1, 0, 1], np.uint8)))
    assert f.p.tolist() == [0, 2] and f.v.tolist() == [10, 30]
    add("filter_plain_paper", "filter", {"a": enc_col(plain), "m": enc_mask(H.PlainMask(np.array([1, 0, 1], np.uint8)))},
        {"col": enc_col(f)}, "proj/tests/test_align.cpp:187-194", {"p": [0, 2], "v": [10, 30]})

    keys = H.RleColumn(np.array([0, 1, 0], np.int64), [0, 2, 5], [1, 4, 8], 9)
    data = H.RleColumn(np.array([3, 3, 3], np.int64), [0, 2, 5], [1, 4, 8], 9)
    ks, vs, ng = ref.group_aggregate([keys], [data, data], ["sum", "count"])
    assert vs[0].tolist() == [18, 9] and vs[1].tolist() == [6, 3]
    add("group_fig6", "group_aggregate", {"keys": [enc_col(keys)], "data": [enc_col(data), enc_col(data)],
                                          "fns": ["sum", "count"]},
        {"keys": [arr(k) for k in ks], "values": [arr(v) for v in vs], "n_groups": ng},
        "proj/tests/test_groupby.cpp:67-88; acceptance.cpp:85-95",
        {"sum": [18, 9], "count": [6, 3]})
    tot = ref.aggregate_all(data, "sum")
    cnt = ref.aggregate_all(data, "count")
    assert (tot, cnt) == (27, 9)
    add("aggregate_all_fig6", "aggregate_all", {"a": enc_col(data), "fn": "sum"}, {"value": scal(tot)},
        "proj/tests/test_groupby.cpp:191-196", {"value": 27})

    m = ref.and_mask(H.RleMask([2], [7], 9), H.RleMask([1, 4, 6], [3, 5, 8], 9))
    assert m.s.tolist() == [2, 4, 6] and m.e.tolist() == [3, 5, 7]
    add("and_rle_paper", "and_mask", {"a": enc_mask(H.RleMask([2], [7], 9)),
                                      "b": enc_mask(H.RleMask([1, 4, 6], [3, 5, 8], 9))},
        {"mask": enc_mask(m)}, "proj/tests/test_logical.cpp:28-33")

    pm = H.PlainMask(np.array([0, 1, 1, 0, 1, 1, 1, 0, 0, 1], np.uint8))
    add("plain_mask_to_rle", "plain_mask_to_rle", {"m": enc_mask(pm)}, {"mask": enc_mask(ref.plain_mask_to_rle(pm))},
        "primitives.cpp:349-360")
    add("plain_mask_to_index", "plain_mask_to_index", {"m": enc_mask(pm)},
        {"mask": enc_mask(ref.plain_mask_to_index(pm))}, "primitives.cpp:362-368")
    gap = H.RleColumn(np.array([5, 6, 7], np.int64), [2, 10, 20], [4, 10, 29], 40)
    add("compact_rle", "compact_rle", {"a": enc_col(gap)}, {"col": enc_col(ref.compact_rle(gap))},
        "proj/tests/test_primitives.cpp:283-298")

    # --- encoders (enc::plain_to_rle / plain_to_rle_index) ----------------------------
    p7 = H.PlainColumn(np.array([0, 0, 0, 0, 1, 1, 1], np.int64))
    r = ref.plain_to_rle(p7)
    assert r.s.tolist() == [0, 4] and r.e.tolist() == [3, 6] and r.v.tolist() == [0, 1]
    add("plain_to_rle_paper", "plain_to_rle", {"a": enc_col(p7)}, {"col": enc_col(r)},
        "proj/tests/test_primitives.cpp:219-226")
    alt = H.PlainColumn(np.arange(64, dtype=np.int64) % 2)
    r = ref.plain_to_rle(alt)
    assert len(r.s) == 64
    add("plain_to_rle_alternating", "plain_to_rle", {"a": enc_col(alt)}, {"col": enc_col(r)},
        "proj/tests/test_primitives.cpp:231-234")
    # narrow storage, centred: run values decoded to the logical type
    nc = H.PlainColumn(np.array([-3, -3, 5, 5, 5, 0, -3], np.int8), H.I64, 1000)
    add("plain_to_rle_narrow_centered", "plain_to_rle", {"a": enc_col(nc)}, {"col": enc_col(ref.plain_to_rle(nc))},
        "primitives.cpp:235-245")
    # storage values that decode equal (wrap at int8) still start separate runs
    wr = H.PlainColumn(np.array([1, 1, 257, 257, 1], np.int64), H.I8)
    r = ref.plain_to_rle(wr)
    assert len(r.s) == 3 and r.v.tolist() == [1, 1, 1]
    add("plain_to_rle_wrap_boundaries", "plain_to_rle", {"a": enc_col(wr)}, {"col": enc_col(r)},
        "kernels.cpp:235-244 (boundaries on storage)")
    p7b = H.PlainColumn(np.array([0, 0, 0, 0, 1, 2, 3], np.int64))
    r = ref.plain_to_rle_index(p7b, 2)
    assert r.runs.s.tolist() == [0] and r.points.p.tolist() == [4, 5, 6]
    add("plain_to_rle_index_paper", "plain_to_rle_index", {"a": enc_col(p7b), "min_run": 2}, {"col": enc_col(r)},
        "proj/tests/test_primitives.cpp:237-245")
    for name, vals, line in (("constant", np.zeros(10, np.int64), "247-250"),
                             ("scattered", np.array([1, 2, 3, 4], np.int64), "252-255")):
        c = H.PlainColumn(vals)
        add(f"plain_to_rle_index_{name}", "plain_to_rle_index", {"a": enc_col(c), "min_run": 2},
            {"col": enc_col(ref.plain_to_rle_index(c, 2))}, f"proj/tests/test_primitives.cpp:{line}")
    erng = np.random.default_rng(10092)
    for it in range(6):
        n = int(erng.integers(50, 600))
        vals = np.repeat(erng.integers(-4, 5, n), erng.integers(1, 6, n))[:n].astype(np.int16)
        c = H.PlainColumn(vals, H.I32, int(erng.integers(-50, 50)) if it % 2 else None)
        add(f"plain_to_rle_rand{it}", "plain_to_rle", {"a": enc_col(c)}, {"col": enc_col(ref.plain_to_rle(c))},
            "seeded")
        mr = 2 + it % 3
        add(f"plain_to_rle_index_rand{it}", "plain_to_rle_index", {"a": enc_col(c), "min_run": mr},
            {"col": enc_col(ref.plain_to_rle_index(c, mr))}, "seeded")

    # --- plain_to_plain_index / choose_encoding / encode / sort_table ----------------
    big = 10_000_000_000
    for name, vals, trim, line in (
            ("wide_outliers", [1, 2, 3, big, big], 0.4, "259-270"),
            ("no_outliers", [5, 6, 7, 8], 0.05, "272-275"),
            ("constant", [9, 9, 9], 0.05, "277-280")):
        c = H.PlainColumn(np.array(vals, np.int64))
        r = ref.plain_to_plain_index(c, trim)
        add(f"plain_to_plain_index_{name}", "plain_to_plain_index", {"a": enc_col(c), "trim": trim},
            {"col": enc_col(r)}, f"proj/tests/test_primitives.cpp:{line}")
    assert ref.plain_to_plain_index(H.PlainColumn(np.array([9, 9, 9], np.int64)), 0.05).base.values.dtype == np.int8
    for it in range(6):
        n = int(erng.integers(100, 2000))
        vals = erng.integers(-30_000, 30_000, n)
        vals[erng.random(n) < 0.02] = erng.integers(1_000_000, 2_000_000_000)
        c = H.PlainColumn(vals.astype(np.int32), H.I64, 7 if it % 2 else None)
        trim = float(erng.choice([0.0, 0.01, 0.05, 0.2]))
        add(f"plain_to_plain_index_rand{it}", "plain_to_plain_index", {"a": enc_col(c), "trim": trim},
            {"col": enc_col(ref.plain_to_plain_index(c, trim))}, "seeded")
    # encoding cascade on small columns (row_threshold lowered so every branch fires)
    cfg = H.Heuristic(row_threshold=64)
    n = 4000
    cascade = {
        "rle": np.repeat(np.arange(4), n // 4),
        "rle_index": np.concatenate([np.repeat(np.arange(2), n // 4), 100 + np.arange(n // 2) % 2]),
        "plain_index": np.where(erng.random(n) < 0.01, 1_500_000_000, erng.integers(-30_000, 30_000, n)),
        "plain_centered": erng.integers(1_000_000, 1_000_100, n),
        "plain": erng.integers(-(1 << 40), 1 << 40, n),
        "float": erng.uniform(0, 1, n),
    }
    for name, vals in cascade.items():
        c = H.PlainColumn(vals)
        ch = ref.choose_encoding(c, cfg)
        add(f"choose_encoding_{name}", "choose_encoding", {"a": enc_col(c), "row_threshold": 64},
            {"choice": list(ch.as_tuple()), "col": enc_col(ref.encode(c, ch))}, "ingest.cpp:217-290")
    assert ref.choose_encoding(H.PlainColumn(np.zeros(100, np.int64))).scheme == H.SCHEME_PLAIN  # test_ingest.cpp:88-92
    k = np.arange(3000) % 3
    cols = [H.PlainColumn(k), H.PlainColumn(np.arange(3000, dtype=np.int32)),
            H.PlainColumn(erng.uniform(-1, 1, 3000))]
    out = ref.sort_table(cols, [0])
    assert len(ref.plain_to_rle(out[0]).s) == 3  # test_ingest.cpp:150-168
    add("sort_table_mod3", "sort_table", {"cols": [enc_col(c) for c in cols], "by": [0]},
        {"cols": [enc_col(c) for c in out]}, "proj/tests/test_ingest.cpp:150-168")
    cols = [H.PlainColumn(erng.integers(0, 4, 500).astype(np.int8), H.I64, 10),
            H.PlainColumn(erng.choice([-0.0, 0.0, 1.5, -2.0], 500)), H.PlainColumn(np.arange(500))]
    add("sort_table_two_keys", "sort_table", {"cols": [enc_col(c) for c in cols], "by": [1, 0]},
        {"cols": [enc_col(c) for c in ref.sort_table(cols, [1, 0])]}, "ingest.cpp:292-344")

    # --- seeded random primitive instances ----------------------------------------
    rng = np.random.default_rng(2506_10092)
    for it in range(12):
        n = int(rng.integers(16, 400))
        s1, e1 = G.random_ranges(rng, n)
        s2, e2 = G.random_ranges(rng, n)
        r = ref.range_intersect(s1, e1, s2, e2)
        add(f"range_intersect_rand{it}", "range_intersect",
            {"s1": s1.tolist(), "e1": e1.tolist(), "s2": s2.tolist(), "e2": e2.tolist()},
            {"s": r[0].tolist(), "e": r[1].tolist(), "idx1": r[2].tolist(), "idx2": r[3].tolist()},
            "seeded; reference test shape test_primitives.cpp:40-74")
        p = G.random_positions(rng, n)
        r = ref.idx_in_rle(p, s1, e1)
        add(f"idx_in_rle_rand{it}", "idx_in_rle", {"p": p.tolist(), "s": s1.tolist(), "e": e1.tolist()},
            {"p_out": r[0].tolist(), "run_of": r[1].tolist(), "idx_of": r[2].tolist()},
            "seeded; test_primitives.cpp:94-105")
        q = G.random_positions(rng, n)
        r = ref.idx_in_idx(p, q)
        add(f"idx_in_idx_rand{it}", "idx_in_idx", {"p1": p.tolist(), "p2": q.tolist()},
            {"p_out": r[0].tolist(), "idx1": r[1].tolist(), "idx2": r[2].tolist()}, "seeded")
        bits = (rng.random(n) < 0.5).astype(np.uint8)
        add(f"plain_mask_to_rle_rand{it}", "plain_mask_to_rle", {"m": enc_mask(H.PlainMask(bits))},
            {"mask": enc_mask(ref.plain_mask_to_rle(H.PlainMask(bits)))}, "seeded")

    # --- operator chains at small scale (C1 / C2 shapes) ----------------------------
    for it in range(4):
        a, b = G.c1_tables(20_000 + 977 * it, 16, 24, seed=100 + it)
        add(f"c1_sum_add_{it}", "sum_binop", {"a": enc_col(a), "b": enc_col(b), "op": "+"},
            {"value": scal(ref.aggregate_all(ref.arith(a, b, "+"), "sum"))},
            "compute::arith + agg::aggregate_all (align.cpp:495-508, groupby.cpp:164-172)")
    for it, variant in enumerate(("rle", "narrow", "rle")):
        n = 30_000 + 1013 * it
        a, b, c = G.c2_tables(n, seed=200 + it, c_variant=variant)
        m = ref.compare_scalar(c, G.C2_K, "<")
        val = ref.aggregate_all(ref.arith(ref.filter(a, m), ref.filter(b, m), "*"), "sum")
        add(f"c2_filtered_sum_{variant}_{it}", "filtered_sum",
            {"a": enc_col(a), "b": enc_col(b), "c": enc_col(c), "k": G.C2_K, "cmp": "<", "op": "*"},
            {"value": scal(val)}, "compare_scalar -> filter x2 -> arith -> aggregate_all (runner.cpp:243-336)")

    with open(OUT, "w") as f:
        json.dump({"generator": "tests/golden/gen_golden.py", "reference": "/root/reference/proj/core (unmodified)",
                   "cases": cases}, f)
    print(f"wrote {len(cases)} cases to {OUT} ({os.path.getsize(OUT)} bytes)")


if __name__ == "__main__":
    main()
