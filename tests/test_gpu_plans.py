"""GPU parity of the device query runner (rq_run_plan, §8f row 4) against
the reference's runq::query::run in Compressed mode (runner.cpp:457-520) on
the same catalog: JSON plans with string and date literals, and / or / not
predicates, projections, inner and semi joins across differently ordered
dictionaries (runner.cpp:198-226 recoding), global and keyed aggregates —
the TPC-H Q1 / Q6 shapes among them, which must take the fused path.
Result rows are compared after the runner's canonical ordering; integers
exact, floats within 1e-9 relative (runner.cpp:394-402)."""
import json

import numpy as np
import pytest

from paper_2506_10092_b200 import host as H
from paper_2506_10092_b200 import queries as Q

pytestmark = pytest.mark.gpu

RF = ["A", "N", "R"]
LS = ["F", "O"]
MODES_L = ["AIR", "RAIL", "SHIP", "TRUCK", "MAIL"]
MODES_T = ["TRUCK", "AIR", "FOB", "MAIL"]
PRIOS = ["5-LOW", "1-URGENT", "3-MEDIUM", "2-HIGH", "4-NOT SPECIFIED"]


def _tables(n, seed):
    rng = np.random.default_rng(seed)
    t = Q.lineitem_q1(n, seed)
    m = max(4, n // 4)
    t["l_orderkey"] = H.PlainColumn(rng.integers(0, m, n).astype(np.int64))
    t["l_shipmode"] = H.PlainColumn(rng.integers(0, len(MODES_L), n).astype(np.int8), H.I64)
    orders = {"o_orderkey": H.PlainColumn(rng.permutation(m).astype(np.int64)),
              "o_orderpriority": H.PlainColumn(rng.integers(0, len(PRIOS), m).astype(np.int64)),
              "o_totalprice": H.PlainColumn(rng.uniform(10, 1000, m))}
    modes = {"m_mode": H.PlainColumn(np.arange(len(MODES_T), dtype=np.int64)),
             "m_weight": H.PlainColumn(np.array([4, 1, 7, 2], np.int64))}
    return t, orders, modes


def _fill(cat, t, orders, modes):
    dicts = {"l_returnflag": RF, "l_linestatus": LS, "l_shipmode": MODES_L}
    for k, c in t.items():
        cat.add_column("lineitem", k, c, dict=dicts.get(k), is_date=(k == "l_shipdate"))
    for k, c in orders.items():
        cat.add_column("orders", k, c, dict=PRIOS if k == "o_orderpriority" else None)
    for k, c in modes.items():
        cat.add_column("modes", k, c, dict=MODES_T if k == "m_mode" else None)


def col(n):
    return {"col": n}


def lit(v):
    return {"lit": v}


def op(o, a, b):
    return {"op": o, "lhs": a, "rhs": b}


def scan(t, cols=None):
    d = {"node": "scan", "table": t}
    if cols:
        d["columns"] = cols
    return d


def agg(fn, name, e=None):
    d = {"fn": fn, "as": name}
    if e is not None:
        d["expr"] = e
    return d


DISC_PRICE = op("*", col("l_extendedprice"), op("-", lit(100), col("l_discount")))
PLANS = {
    "q1": ({"node": "group_agg", "keys": ["l_returnflag", "l_linestatus"],
            "aggs": [agg("sum", "sum_qty", col("l_quantity")), agg("sum", "sum_base", col("l_extendedprice")),
                     agg("sum", "sum_disc_price", DISC_PRICE),
                     agg("sum", "sum_charge", op("*", DISC_PRICE, op("+", col("l_tax"), lit(100)))),
                     agg("avg", "avg_qty", col("l_quantity")), agg("avg", "avg_price", col("l_extendedprice")),
                     agg("avg", "avg_disc", col("l_discount")), agg("count", "count_order")],
            "input": {"node": "filter", "pred": op("<=", col("l_shipdate"), lit("1998-09-02")),
                      "input": scan("lineitem")}}, True),
    "q6": ({"node": "group_agg", "aggs": [agg("sum", "revenue", op("*", col("l_extendedprice"), col("l_discount")))],
            "input": {"node": "filter",
                      "pred": op("and", op("and", op(">=", col("l_shipdate"), lit("1994-01-01")),
                                            op("<", col("l_shipdate"), lit("1995-01-01"))),
                                 op("and", op("and", op(">=", col("l_discount"), lit(5)),
                                               op("<=", col("l_discount"), lit(7))),
                                    op("<", col("l_quantity"), lit(24)))),
                      "input": scan("lineitem")}}, True),
    "in_list_reversed": ({"node": "group_agg", "keys": ["l_linestatus"],
                          "aggs": [agg("count", "n"), agg("sum", "q", col("l_quantity")),
                                   agg("avg", "p", op("/", col("l_extendedprice"), lit(2.5)))],
                          "input": {"node": "filter",
                                    "pred": op("and", op("or", op("==", col("l_returnflag"), lit("R")),
                                                         op("==", col("l_returnflag"), lit("A"))),
                                               op(">", lit(40), col("l_quantity"))),
                                    "input": scan("lineitem")}}, True),
    "not_pred": ({"node": "group_agg", "keys": ["l_returnflag"],
                  "aggs": [agg("count", "n"), agg("max", "mx", col("l_quantity"))],
                  "input": {"node": "filter",
                            "pred": {"op": "not", "arg": op("<", col("l_quantity"), lit(10))},
                            "input": scan("lineitem")}}, False),
    "project": ({"node": "group_agg", "keys": ["l_linestatus"],
                 "aggs": [agg("sum", "v", col("v")), agg("var", "w", col("v"))],
                 "input": {"node": "project",
                           "exprs": [{"expr": col("l_linestatus"), "as": "l_linestatus"},
                                     {"expr": op("*", col("l_extendedprice"), lit(2)), "as": "v"}],
                           "input": scan("lineitem")}}, False),
    "inner_join": ({"node": "group_agg", "keys": ["o_orderpriority"],
                    "aggs": [agg("count", "n"), agg("sum", "q", col("l_quantity")),
                             agg("sum", "t", col("o_totalprice"))],
                    "input": {"node": "join", "on": {"left": "l_orderkey", "right": "o_orderkey"},
                              "left": scan("lineitem", ["l_orderkey", "l_quantity"]),
                              "right": scan("orders")}}, False),
    "semi_join_recode": ({"node": "group_agg", "keys": ["l_shipmode"],
                          "aggs": [agg("count", "n"), agg("min", "lo", col("l_extendedprice"))],
                          "input": {"node": "join", "kind": "semi", "on": {"left": "l_shipmode", "right": "m_mode"},
                                    "left": scan("lineitem"), "right": scan("modes")}}, False),
    "global_count": ({"node": "group_agg", "aggs": [agg("count", "n"), agg("sum", "s", col("l_tax"))],
                      "input": scan("lineitem")}, False),
}


def _canon(res):
    names = list(res)
    n = len(res[names[0]]) if names else 0
    order = sorted(range(n), key=lambda i: tuple((0, 0.0) if isinstance(res[c][i], float) and np.isnan(res[c][i])
                                                 else (1, float(res[c][i])) for c in names))
    return {c: np.asarray(res[c])[order] for c in names}


@pytest.mark.parametrize("n", [5_000, 400_000])
@pytest.mark.parametrize("name", sorted(PLANS))
def test_plan_vs_reference(rq, ref, name, n):
    from oracle.refpy import RefCatalog
    plan, must_fuse = PLANS[name]
    t, orders, modes = _tables(n, 11 + n % 7)
    dcat, rcat = rq.Catalog(), RefCatalog(ref)
    _fill(dcat, t, orders, modes)
    _fill(rcat, t, orders, modes)
    text = json.dumps({"plan": plan})
    got, rows, fused = dcat.run_plan(text)
    want = rcat.run_plan(text)
    assert list(got) == list(want), (list(got), list(want))
    g, w = _canon(got), _canon(want)
    for c in want:
        a, b = g[c], w[c]
        assert len(a) == len(b), f"{c}: {len(a)} rows != {len(b)}"
        if np.issubdtype(b.dtype, np.floating) or np.issubdtype(a.dtype, np.floating):
            a, b = a.astype(np.float64), b.astype(np.float64)
            tol = 1e-9 * np.maximum(1.0, np.maximum(np.abs(a), np.abs(b)))
            assert np.all((np.abs(a - b) <= tol) | (np.isnan(a) & np.isnan(b))), c
        else:
            assert np.array_equal(a.astype(np.int64), b.astype(np.int64)), c
    if must_fuse:
        assert fused == 1, f"{name}: expected the fused GroupAgg path"


def test_plan_errors_match_reference(rq, ref):
    """Unknown columns and string literals against non-string columns raise."""
    from paper_2506_10092_b200._lib import RqError
    t, orders, modes = _tables(1000, 3)
    dcat = rq.Catalog()
    _fill(dcat, t, orders, modes)
    bad = {"node": "group_agg", "aggs": [agg("count", "n")],
           "input": {"node": "filter", "pred": op("==", col("l_quantity"), lit("x")), "input": scan("lineitem")}}
    with pytest.raises(RqError):
        dcat.run_plan(json.dumps(bad))
    with pytest.raises(RqError):
        dcat.run_plan(json.dumps({"node": "scan", "table": "nope"}))


# ---- random plans: predicate trees x keys x expression aggregates ------------------

NUM_COLS = ["l_quantity", "l_extendedprice", "l_discount", "l_tax"]


def _rand_cmp(rng):
    c = str(rng.choice(NUM_COLS + ["l_shipdate", "l_returnflag", "l_linestatus", "l_shipmode"]))
    o = str(rng.choice(["<", "<=", "==", "!=", ">=", ">"]))
    if c == "l_shipdate":
        v = lit(f"199{int(rng.integers(2, 9))}-0{int(rng.integers(1, 10))}-1{int(rng.integers(0, 10))}")
    elif c == "l_returnflag":
        v = lit(str(rng.choice(RF + ["Z"])))  # absent strings resolve to code -1
    elif c == "l_linestatus":
        v = lit(str(rng.choice(LS)))
    elif c == "l_shipmode":
        v = lit(str(rng.choice(MODES_L)))
    elif c == "l_extendedprice":
        v = lit(float(rng.uniform(900, 100000)))
    else:
        v = lit(int(rng.integers(0, 51)))
    return op(o, v, col(c)) if rng.random() < 0.2 else op(o, col(c), v)


def _rand_pred(rng, depth):
    r = rng.random()
    if depth == 0 or r < 0.4:
        return _rand_cmp(rng)
    if r < 0.55:
        return {"op": "not", "arg": _rand_pred(rng, depth - 1)}
    return op(str(rng.choice(["and", "or"])), _rand_pred(rng, depth - 1), _rand_pred(rng, depth - 1))


def _rand_expr(rng, depth=2):
    r = rng.random()
    if depth == 0 or r < 0.35:
        return col(str(rng.choice(NUM_COLS)))
    if r < 0.6:
        k = lit(int(rng.integers(1, 100))) if rng.random() < 0.6 else lit(float(rng.uniform(0.5, 3.0)))
        o = str(rng.choice(["+", "-", "*"]))
        return op(o, k, _rand_expr(rng, depth - 1)) if rng.random() < 0.3 else op(o, _rand_expr(rng, depth - 1), k)
    if r < 0.7:
        return op("/", _rand_expr(rng, depth - 1), lit(float(rng.uniform(0.5, 4.0))))
    return op(str(rng.choice(["+", "-", "*"])), _rand_expr(rng, depth - 1), _rand_expr(rng, depth - 1))


@pytest.mark.parametrize("seed", range(80))
def test_random_plans_vs_reference(rq, ref, seed):
    """Random filter trees (and / or / not over every column kind, reversed
    literals, absent dictionary strings), random key sets and random
    expression aggregates: the device runner (fused or chain, whichever the
    plan takes) against the reference runner."""
    from oracle.refpy import RefCatalog
    rng = np.random.default_rng(900 + seed)
    n = int(rng.integers(2_000, 60_000))
    t, orders, modes = _tables(n, 500 + seed)
    keys = [k for k in ("l_returnflag", "l_linestatus", "l_shipmode") if rng.random() < 0.35]
    aggs = [agg("count", "n")]
    for i in range(int(rng.integers(1, 5))):
        aggs.append(agg(str(rng.choice(["sum", "avg", "min", "max"])), f"a{i}", _rand_expr(rng)))
    plan = {"node": "group_agg", "aggs": aggs,
            "input": {"node": "filter", "pred": _rand_pred(rng, 3), "input": scan("lineitem")}}
    if keys:
        plan["keys"] = keys
    dcat, rcat = rq.Catalog(), RefCatalog(ref)
    _fill(dcat, t, orders, modes)
    _fill(rcat, t, orders, modes)
    text = json.dumps({"plan": plan})
    got, rows, fused = dcat.run_plan(text)
    want = rcat.run_plan(text)
    assert list(got) == list(want), (list(got), list(want))
    g, w = _canon(got), _canon(want)
    for c in want:
        a, b = g[c], w[c]
        assert len(a) == len(b), f"{c}: {len(a)} rows != {len(b)} ({text})"
        if np.issubdtype(b.dtype, np.floating) or np.issubdtype(a.dtype, np.floating):
            a, b = a.astype(np.float64), b.astype(np.float64)
            tol = 1e-9 * np.maximum(1.0, np.maximum(np.abs(a), np.abs(b)))
            with np.errstate(invalid="ignore"):  # equal infinities (empty MIN / MAX sentinels) subtract to NaN
                ok = (a == b) | (np.abs(a - b) <= tol) | (np.isnan(a) & np.isnan(b))
            assert np.all(ok), f"{c}: {text}"
        else:
            assert np.array_equal(a.astype(np.int64), b.astype(np.int64)), f"{c}: {text}"


@pytest.mark.parametrize("seed", range(24))
def test_random_join_plans_vs_reference(rq, ref, seed):
    """Random filtered inner / semi joins (lineitem ⋈ orders on the key,
    lineitem ⋉ modes across differently ordered dictionaries) under random
    keys and aggregates, against the reference runner."""
    from oracle.refpy import RefCatalog
    rng = np.random.default_rng(4000 + seed)
    n = int(rng.integers(2_000, 40_000))
    t, orders, modes = _tables(n, 700 + seed)
    left = {"node": "filter", "pred": _rand_pred(rng, 2), "input": scan("lineitem")}
    if rng.random() < 0.5:
        j = {"node": "join", "on": {"left": "l_orderkey", "right": "o_orderkey"}, "left": left,
             "right": scan("orders")}
        keys = ["o_orderpriority"] if rng.random() < 0.6 else []
        pool = NUM_COLS + ["o_totalprice"]
    else:
        j = {"node": "join", "kind": "semi", "on": {"left": "l_shipmode", "right": "m_mode"}, "left": left,
             "right": {"node": "filter", "pred": op(">", col("m_weight"), lit(int(rng.integers(0, 6)))),
                       "input": scan("modes")}}
        keys = ["l_shipmode"] if rng.random() < 0.6 else []
        pool = NUM_COLS
    aggs = [agg("count", "n")]
    for i in range(int(rng.integers(1, 4))):
        e = col(str(rng.choice(pool)))
        if rng.random() < 0.5:
            e = op(str(rng.choice(["+", "*", "-"])), e, lit(int(rng.integers(1, 9))))
        aggs.append(agg(str(rng.choice(["sum", "avg", "min", "max"])), f"a{i}", e))
    plan = {"node": "group_agg", "aggs": aggs, "input": j}
    if keys:
        plan["keys"] = keys
    dcat, rcat = rq.Catalog(), RefCatalog(ref)
    _fill(dcat, t, orders, modes)
    _fill(rcat, t, orders, modes)
    text = json.dumps({"plan": plan})
    got, rows, fused = dcat.run_plan(text)
    want = rcat.run_plan(text)
    assert list(got) == list(want), (list(got), list(want))
    g, w = _canon(got), _canon(want)
    for c in want:
        a, b = g[c], w[c]
        assert len(a) == len(b), f"{c}: {len(a)} rows != {len(b)} ({text})"
        if np.issubdtype(b.dtype, np.floating) or np.issubdtype(a.dtype, np.floating):
            a, b = a.astype(np.float64), b.astype(np.float64)
            tol = 1e-9 * np.maximum(1.0, np.maximum(np.abs(a), np.abs(b)))
            with np.errstate(invalid="ignore"):
                ok = (a == b) | (np.abs(a - b) <= tol) | (np.isnan(a) & np.isnan(b))
            assert np.all(ok), f"{c}: {text}"
        else:
            assert np.array_equal(a.astype(np.int64), b.astype(np.int64)), f"{c}: {text}"


def _gapped_rle(rng, n, L, lo, hi):
    e = np.cumsum(rng.integers(1, 2 * L, n // L + 2))
    e = e[e < n - 1]
    e = np.append(e, n - 1).astype(np.int64)
    s = np.concatenate([[0], e[:-1] + 1]).astype(np.int64)
    keep = rng.random(len(s)) > 0.35
    return H.RleColumn(rng.integers(lo, hi + 1, int(keep.sum())).astype(np.int64), s[keep], e[keep], n)


@pytest.mark.parametrize("seed", [1, 2])
def test_plan_coverage_rules_with_gapped_columns(rq, ref, seed):
    """Catalog columns with gaps: the runner aligns keys with ALL data jointly
    — for count(*) through the scan's first column — and aggregates each
    expression over its own coverage when there are no keys
    (runner.cpp:302-336). The fused pass must not be taken where its shared
    segment table would differ (gapped first column, no-key
    expressions over differently gapped columns)."""
    from oracle.refpy import RefCatalog
    rng = np.random.default_rng(seed)
    n = 60_000
    t = {"g1": _gapped_rle(rng, n, 300, 0, 50), "key": _gapped_rle(rng, n, 2000, 0, 4) if seed == 2 else
         H.RleColumn(*_full_rle(rng, n, 2000, 0, 4), n),
         "a": _gapped_rle(rng, n, 40, -20, 20), "b": _gapped_rle(rng, n, 70, 1, 9),
         "p": H.PlainColumn(rng.integers(-100, 100, n).astype(np.int16), H.I64)}
    plans = [
        {"node": "group_agg", "keys": ["key"], "aggs": [agg("count", "n"), agg("sum", "s", col("p"))],
         "input": scan("t")},
        {"node": "group_agg", "aggs": [agg("sum", "sa", col("a")), agg("sum", "sb", col("b")),
                                       agg("avg", "ap", col("p"))], "input": scan("t")},
        {"node": "group_agg", "keys": ["key"], "aggs": [agg("count", "n"), agg("sum", "s", col("a"))],
         "input": {"node": "filter", "pred": op("<", col("b"), lit(6)), "input": scan("t")}},
    ]
    dcat, rcat = rq.Catalog(), RefCatalog(ref)
    for k, c in t.items():
        dcat.add_column("t", k, c)
        rcat.add_column("t", k, c)
    for plan in plans:
        text = json.dumps({"plan": plan})
        got, rows, fused = dcat.run_plan(text)
        want = rcat.run_plan(text)
        g, w = _canon(got), _canon(want)
        assert list(got) == list(want)
        for c in want:
            a, b = g[c].astype(np.float64), w[c].astype(np.float64)
            assert len(a) == len(b), (plan, c)
            tol = 1e-9 * np.maximum(1.0, np.maximum(np.abs(a), np.abs(b)))
            assert np.all((np.abs(a - b) <= tol) | (np.isnan(a) & np.isnan(b))), (plan, c)


def _full_rle(rng, n, L, lo, hi):
    e = np.cumsum(rng.integers(1, 2 * L, n // L + 2))
    e = e[e < n - 1]
    e = np.append(e, n - 1).astype(np.int64)
    s = np.concatenate([[0], e[:-1] + 1]).astype(np.int64)
    return rng.integers(lo, hi + 1, len(s)).astype(np.int64), s, e
