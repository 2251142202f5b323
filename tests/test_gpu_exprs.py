"""GPU parity of the fused Filter → expressions → GroupAgg path (K12,
rq_group_aggregate_exprs) against the reference library running the
runner's operator chain (runner.cpp:243-336) on the same inputs: the C4
Q1 / Q6 plans, the C5 plan, and randomized expression / mask / key shapes
(narrow centred plain, f64, RLE operands, Plain+Index, scalar ops both ways,
int ÷0). Integer results bit-exact; f64 within 1e-9 relative."""
import numpy as np
import pytest

from helpers import assert_array, assert_scalar
from paper_2506_10092_b200 import datagen as G
from paper_2506_10092_b200 import host as H
from paper_2506_10092_b200 import queries as Q
from paper_2506_10092_b200._lib import RqError

pytestmark = pytest.mark.gpu


def ref_api(ref):
    from oracle.refpy import RefAPI
    return RefAPI(ref)


@pytest.mark.parametrize("n", [1000, 300_000, 3_000_000])
def test_q1_fused_vs_reference(rq, ref, n, row_kernel):
    t = Q.lineitem_q1(n, seed=n + 1)
    (ks, vs, ng), fused = Q.q1_fused(rq, t)
    assert fused
    wk, wv, wng = Q.q1(ref_api(ref), t)
    assert ng == wng
    for g, w in zip(ks + vs, wk + wv):
        assert_array(g, w)


@pytest.mark.parametrize("n", [1000, 300_000, 3_000_000])
def test_q6_fused_vs_reference(rq, ref, n):
    t = Q.lineitem_q6(n, seed=n)
    got, fused = Q.q6_fused(rq, t)
    assert fused
    assert_scalar(got, Q.q6(ref_api(ref), t), "q6")


@pytest.mark.parametrize("n", [5_000, 400_000])
def test_c5_fused_vs_reference(rq, ref, n):
    t = Q.production_table(n, seed=n)
    (ks, vs, ng), fused = Q.c5_fused(rq, t)
    assert fused
    wk, wv, wng = Q.c5_query(ref_api(ref), t)
    assert ng == wng
    for g, w in zip(ks + vs, wk + wv):
        assert_array(g, w)


def _rle(rng, n, L, lo, hi, gaps=False):
    e = G.run_ends(n, L, rng)
    s = np.concatenate([[0], e[:-1] + 1])
    if gaps:
        keep = rng.random(len(s)) > 0.3
        s, e = s[keep], e[keep]
    return H.RleColumn(rng.integers(lo, hi + 1, len(s)).astype(np.int64), s.astype(np.int64), e.astype(np.int64), n)


def _chain(ref, mask, keys, exprs, fns):
    """The runner's chain on the reference library for X expressions."""
    F = (lambda c: ref.filter(c, mask)) if mask is not None else (lambda c: c)
    data = []
    for x in exprs:
        if not x.terms:
            data.append(F(keys[0]))
            continue

        def term(tm):
            c, op, rev, k = tm
            return ref.arith_scalar(F(c), k, H.BINOP_NAMES.get(op, op), rev) if op != -1 else F(c)
        v = term(x.terms[0])
        for tm, op in zip(x.terms[1:], x.ops):
            v = ref.arith(v, term(tm), op)
        data.append(v)
    kf = [ref.normalize_basic(F(k)) for k in keys]
    return ref.group_aggregate(kf, [ref.normalize_basic(d) for d in data], fns)


@pytest.fixture(params=["generated", "interpreted"])
def row_kernel(request, monkeypatch):
    """Both K12 row kernels: the NVRTC-specialised one and the interpreted one."""
    if request.param == "interpreted":
        monkeypatch.setenv("RQ_NO_JIT", "1")
    else:
        monkeypatch.delenv("RQ_NO_JIT", raising=False)
    return request.param


@pytest.mark.parametrize("inst", range(8))
def test_random_expressions_vs_reference(rq, ref, inst, row_kernel):
    rng = np.random.default_rng(300 + inst)
    X = rq.X
    n = int(rng.integers(1000, 400_000))
    k1 = _rle(rng, n, int(rng.integers(50, 5000)), 0, 6)
    k2 = _rle(rng, n, int(rng.integers(500, 50_000)), 10, 12, gaps=bool(inst % 3 == 2))
    p8 = H.PlainColumn(rng.integers(-100, 101, n).astype(np.int8), H.I64, int(rng.integers(-50, 50)))
    p16 = H.PlainColumn(rng.integers(-3000, 3001, n).astype(np.int16), H.I32, None)
    pf = H.PlainColumn(rng.uniform(-50, 50, n))
    r = _rle(rng, n, 40, -9, 9)
    pi = Q._plain_index(rng, n, 0.02)
    mcol = _rle(rng, n, 200, 0, 9)
    mask = rq.compute.compare_scalar(mcol, 6, "<") if inst % 2 == 0 else None
    hmask = ref.compare_scalar(mcol, 6, "<") if mask is not None else None
    exprs = [X.col(p8), X.col(pf).arith(X.col(p16).scalar(7, "-", True), "*"),
             X.col(p8).arith(X.col(r), "+").arith(X.col(p16).scalar(3, "*"), "-"),
             X.col(r).scalar(2.5, "*"), X.col(pi), X.count(), X.col(p16), X.col(pf)]
    fns = ["sum", "sum", "sum", "avg", "sum", "count", "avg", "avg"]
    keys = [k1] if inst % 4 < 2 else [k1, k2]
    ks, vs, ng, fused = rq.agg.group_aggregate_exprs(mask, keys, exprs, fns)
    assert fused
    wk, wv, wng = _chain(ref, hmask, keys, exprs, fns)
    assert ng == wng
    for g, w in zip(ks + vs, wk + wv):
        assert_array(g, w)


def test_global_aggregate_and_division(rq, ref, row_kernel):
    rng = np.random.default_rng(9)
    X = rq.X
    n = 200_000
    a = H.PlainColumn(rng.integers(-500, 500, n).astype(np.int16), H.I64, None)
    b = _rle(rng, n, 30, 1, 9)
    ks, vs, ng, fused = rq.agg.group_aggregate_exprs(None, [], [X.col(a).arith(X.col(b), "/"), X.count()],
                                                     ["sum", "count"])
    assert fused and ng == 1
    q = ref.arith(a, b, "/")
    assert int(vs[0][0]) == ref.aggregate_all(q, "sum")
    assert int(vs[1][0]) == n
    bz = H.RleColumn(np.zeros(len(b.v), np.int64), b.s, b.e, n)
    with pytest.raises(RqError):
        rq.agg.group_aggregate_exprs(None, [], [X.col(a).arith(X.col(bz), "/")], ["sum"])


def test_unfusable_shapes_fall_back_to_chain(rq, ref):
    """Index operands / MIN take the operator chain — same results."""
    rng = np.random.default_rng(10)
    X = rq.X
    n = 50_000
    k = _rle(rng, n, 300, 0, 4)
    idx = G.sparse_index(n, 0.05, 3)
    p = H.PlainColumn(rng.integers(0, 100, n).astype(np.int64))
    ks, vs, ng, fused = rq.agg.group_aggregate_exprs(None, [k], [X.col(p), X.col(p)], ["sum", "max"])
    assert not fused
    wk, wv, wng = _chain(ref, None, [k], [X.col(p), X.col(p)], ["sum", "max"])
    assert ng == wng
    for g, w in zip(ks + vs, wk + wv):
        assert_array(g, w)
    _, vs, _, fused = rq.agg.group_aggregate_exprs(None, [k], [X.col(idx)], ["sum"])
    assert not fused


def _ref_where_mask(ref, where):
    m = None
    for col, op, k in where:
        if op == "in":
            c = None
            for x in k:
                e = ref.compare_scalar(col, x, "==")
                c = e if c is None else ref.or_mask(c, e)
        else:
            c = ref.compare_scalar(col, k, op)
        m = c if m is None else ref.and_mask(m, c)
    return m


@pytest.mark.parametrize("inst", range(6))
def test_where_pushdown_vs_reference(rq, ref, inst, row_kernel):
    """WHERE conjuncts evaluated per run segment (no mask) == the runner's
    compare_scalar / or_mask / and_mask mask followed by the chain."""
    rng = np.random.default_rng(900 + inst)
    X = rq.X
    n = int(rng.integers(5_000, 500_000))
    k1 = _rle(rng, n, int(rng.integers(100, 20_000)), 0, 5)
    p1 = _rle(rng, n, 80, 0, 30, gaps=bool(inst % 2))
    p2 = _rle(rng, n, 900, -5, 5)
    pf = H.PlainColumn(rng.uniform(0, 10, n))
    p8 = H.PlainColumn(rng.integers(-100, 101, n).astype(np.int8), H.I64, 3)
    where = [(p1, "in", [1, 7, 12, 29]), (p2, ">=", -2), (p2, "<", 4.5)]
    if inst >= 3:
        where = where[1:] + [(p1, "!=", 3)]
    exprs = [X.col(pf).arith(X.col(p8), "*"), X.col(p8), X.count(), X.col(p2).scalar(2, "*")]
    fns = ["sum", "avg", "count", "sum"]
    keys = [k1] if inst % 3 else []
    ks, vs, ng, fused = rq.agg.group_aggregate_exprs(None, keys, exprs, fns, where=where)
    assert fused
    hm = _ref_where_mask(ref, where)
    if keys:
        wk, wv, wng = _chain(ref, hm, keys, exprs, fns)
        assert ng == wng
        for g, w in zip(ks + vs, wk + wv):
            assert_array(g, w)
    else:
        for i, (x, fn) in enumerate(zip(exprs, fns)):
            if not x.terms:
                want = ref.aggregate_all(ref.filter(p2, hm), "count")
            else:
                def term(tm):
                    c, op, rev, kk = tm
                    return ref.arith_scalar(ref.filter(c, hm), kk, op, rev) if op != -1 else ref.filter(c, hm)
                v = term(x.terms[0])
                for tm, op in zip(x.terms[1:], x.ops):
                    v = ref.arith(v, term(tm), op)
                want = ref.aggregate_all(v, fn)
            got = vs[i][0]
            assert_scalar(float(got) if isinstance(want, float) else int(got), want, f"expr {i}")


_FOLD_CASES = [
    # conjuncts on one integer run column, folded to interval ∩ value set
    [("p1", "in", [1, 7.0, 7.5, 12, 29]), ("p1", "in", [7, 12, 13]), ("p2", ">", -2.5), ("p2", "<=", 3.9)],
    [("p1", "==", 7.0), ("p2", "!=", 0), ("p2", "!=", 99)],
    [("p1", "==", 7.5)],                                   # never equal: empty result
    [("p1", ">=", 20), ("p1", "<", 10)],                    # contradictory interval
    [("p1", "<", 1e300), ("p2", ">", -1e300)],              # out-of-range literals: interpreted
    [("p1", "!=", 3), ("p1", "!=", 4), ("p1", "in", [3, 4, 5, 6])],
    [("pf", "<", 5.0), ("p1", ">=", 10)],                   # float run values: interpreted
    [("p2", ">=", -9223372036854775808), ("p1", "<=", 9223372036854775807)],
]


@pytest.mark.parametrize("case", range(len(_FOLD_CASES)))
def test_where_folded_conjuncts_vs_reference(rq, ref, case):
    """The segment table folds a list's integer conjuncts into one interval
    and value set: float literals (integral or not), NE exclusions, IN lists
    intersected, empty and unbounded ranges == compare_scalar's masks."""
    rng = np.random.default_rng(1200 + case)
    X = rq.X
    n = 200_000
    cols = {"p1": _rle(rng, n, 80, 0, 30), "p2": _rle(rng, n, 900, -5, 5)}
    pf = _rle(rng, n, 500, 0, 10)
    cols["pf"] = H.RleColumn(pf.v.astype(np.float64) + 0.25, pf.s, pf.e, n)
    k1 = _rle(rng, n, 5_000, 0, 5)
    v = H.PlainColumn(rng.integers(-100, 101, n).astype(np.int64))
    where = [(cols[c], op, k) for c, op, k in _FOLD_CASES[case]]
    exprs, fns = [X.col(v), X.count()], ["sum", "count"]
    ks, vs, ng, fused = rq.agg.group_aggregate_exprs(None, [k1], exprs, fns, where=where)
    assert fused
    wk, wv, wng = _chain(ref, _ref_where_mask(ref, where), [k1], exprs, fns)
    assert ng == wng
    for g, w in zip(ks + vs, wk + wv):
        assert_array(g, w)


def test_where_on_plain_column_falls_back_to_mask(rq, ref):
    """A conjunct on a plain column cannot be evaluated per run segment: the
    call builds the runner's mask and still fuses the aggregation."""
    rng = np.random.default_rng(77)
    X = rq.X
    n = 200_000
    k = _rle(rng, n, 500, 0, 4)
    p = H.PlainColumn(rng.integers(0, 100, n).astype(np.int16), H.I64, None)
    r = _rle(rng, n, 60, 0, 9)
    where = [(p, "<", 40), (r, ">", 2)]
    ks, vs, ng, fused = rq.agg.group_aggregate_exprs(None, [k], [X.col(p), X.count()], ["sum", "count"],
                                                     where=where)
    assert fused
    wk, wv, wng = _chain(ref, _ref_where_mask(ref, where), [k], [X.col(p), X.count()], ["sum", "count"])
    assert ng == wng
    for g, w in zip(ks + vs, wk + wv):
        assert_array(g, w)


@pytest.mark.parametrize("n", [1003, 77_777])
def test_plain_divisor_zeros_only_on_dropped_rows(rq, ref, n, row_kernel):
    """SUM(a / b) with a Plain i64 divisor that is 0 only on rows the WHERE
    drops (and n % 8 != 0, so the last window has padding rows): the reference
    filters first and divides only kept rows (align.cpp:290-305, :755-771), so
    no error; a zero on a kept row still raises."""
    rng = np.random.default_rng(n)
    X = rq.X
    k = _rle(rng, n, 97, 0, 3)
    mcol = _rle(rng, n, 13, 0, 9)
    keep = np.zeros(n, bool)
    for s, e, v in zip(mcol.s, mcol.e, mcol.v):
        keep[s:e + 1] = v < 5
    bv = rng.integers(1, 50, n).astype(np.int64)
    bv[~keep] = 0
    a = H.PlainColumn(rng.integers(-1000, 1000, n).astype(np.int64))
    b = H.PlainColumn(bv)
    mask = rq.compute.compare_scalar(mcol, 5, "<")
    hmask = ref.compare_scalar(mcol, 5, "<")
    # a / b and the reversed scalar 1000 / b both divide by b = 0 on dropped rows
    exprs = [X.col(a).arith(X.col(b), "/"), X.col(b).scalar(1000, "/", True), X.count()]
    fns = ["sum", "sum", "count"]
    ks, vs, ng, fused = rq.agg.group_aggregate_exprs(mask, [k], exprs, fns)
    assert fused
    wk, wv, wng = _chain(ref, hmask, [k], exprs, fns)
    assert ng == wng
    for g, w in zip(ks + vs, wk + wv):
        assert_array(g, w)
    # no WHERE: the zeros are on counted rows now -> integer division by zero
    with pytest.raises(RqError):
        rq.agg.group_aggregate_exprs(None, [k], [X.col(a).arith(X.col(b), "/")], ["sum"])
