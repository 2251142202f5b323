"""TPC-H-style Q6 / Q1 over a synthetic lineitem (BASELINE config C4).

The reference has no TPC-H generator or Q1 plan;
its query runner evaluates a plan as: predicate masks (compare_scalar per
literal, and_mask per conjunction, runner.cpp:114-193) → Filter applies the
mask to EVERY scanned column (runner.cpp:243-252) → GroupAgg evaluates each
aggregate expression with binary/scalar ops, normalizes keys and inputs and
calls aggregate_all (no keys) or group_aggregate (runner.cpp:302-336).
``q6`` / ``q1`` restate those plans against an operator API object ``api``
with the reference's namespaces (``api.compute``, ``api.masks``,
``api.agg``): the device path passes ``paper_2506_10092_b200.runq``; tests and
the bench's reference arm pass an adapter over the reference library, so both
sides run the same operator sequence.

Synthetic lineitem: returnflag {A,N,R} → codes 0..2,
linestatus {F,O} → 0..1, shipdate days since 1970 in [8036, 10561], quantity
1..50, discount 0..10 and tax 0..8 in hundredths (ints; the paper keeps
decimals as floats, here hundredths keep the sums exact), extendedprice f64.
Tables are sorted per query as in the paper's Table 7:
Q1 by (returnflag, linestatus, shipdate, quantity), Q6 by (quantity,
discount, shipdate); low-cardinality sort keys are RLE, discount/tax
plain-centered i8, price plain f64. At SF100 that is exactly what the
device's choose_encoding (ingest.cpp:217-271; itself checked against the
reference's) picks for each decoded column — tests/test_gpu_encode_choice.py
runs it on the full 600M-row columns. (At SF1-SF10 the heuristic picks
plain-centered for some sort keys whose runs are still short, e.g. Q6's
shipdate below ~SF50; the generator keeps the SF100 encodings at every
scale so the plan shape is the same.)
"""
from __future__ import annotations

import numpy as np

from . import host as H
from .datagen import cut, part_range, positional, positional_column, run_ends

ROWS_PER_SF = 6_000_000
SHIP_LO, SHIP_HI = 8036, 10561      # 1992-01-02 .. 1998-12-01
Q6_LO, Q6_HI = 8766, 9131           # [1994-01-01, 1995-01-01)
Q1_CUTOFF = 10471                   # 1998-09-02
DISC_CENTER, TAX_CENTER = 5, 4      # choose_encoding's plain-centered centres (mid-range)


def _rle_from_sorted(vals: np.ndarray, total: int) -> H.RleColumn:
    """RLE of a sorted-by-key value array (plain_to_rle, primitives.cpp:223-250)."""
    n = len(vals)
    if n == 0:
        return H.RleColumn(np.empty(0, vals.dtype), [], [], total)
    brk = np.nonzero(vals[1:] != vals[:-1])[0]
    s = np.concatenate([[0], brk + 1]).astype(np.int64)
    e = np.concatenate([brk, [n - 1]]).astype(np.int64)
    return H.RleColumn(vals[s], s, e, total)


def _rle_from_counts(values: np.ndarray, counts: np.ndarray, total: int) -> H.RleColumn:
    """RLE of consecutive groups (value, count), empty groups dropped and equal
    neighbours merged (plain_to_rle of the sorted column, primitives.cpp:223-250)."""
    keep = counts > 0
    values, counts = values[keep], counts[keep]
    if len(values):
        brk = np.concatenate([[True], values[1:] != values[:-1]])
        grp = np.cumsum(brk) - 1
        counts = np.bincount(grp, weights=counts).astype(np.int64)
        values = values[brk]
    e = np.cumsum(counts) - 1
    s = e - counts + 1
    return H.RleColumn(values.astype(np.int64), s.astype(np.int64), e.astype(np.int64), total)


def lineitem_q6(n: int, seed: int = 42, part=None, slicer=None):
    """Lineitem sorted by (quantity, discount, shipdate); the sorted key
    columns are generated directly as runs (multinomial group sizes) over the
    whole table and cut to this part's rows (snapped to shipdate's runs);
    price is positional (datagen.positional)."""
    rng = np.random.default_rng(seed)
    days = np.arange(SHIP_LO, SHIP_HI + 1, dtype=np.int64)
    qc = rng.multinomial(n, np.full(50, 1 / 50))
    dvals, dcounts, svals, scounts = [], [], [], []
    for q in range(50):
        dc = rng.multinomial(qc[q], np.full(11, 1 / 11))
        dvals.append(np.arange(11))
        dcounts.append(dc)
        for d in range(11):
            sc = rng.multinomial(dc[d], np.full(len(days), 1 / len(days)))
            svals.append(days)
            scounts.append(sc)
    ship = _rle_from_counts(np.concatenate(svals), np.concatenate(scounts), n)
    lo, hi = part_range(n, part, ship)
    price = positional(n, seed + 1, lo, hi, lambda r, m: r.uniform(900.0, 105000.0, m), np.float64)
    return {
        "l_quantity": cut(_rle_from_counts(np.arange(1, 51), qc, n), lo, hi, slicer),
        "l_discount": cut(_rle_from_counts(np.concatenate(dvals), np.concatenate(dcounts), n), lo, hi, slicer),
        "l_shipdate": cut(ship, lo, hi, slicer),
        "l_extendedprice": H.PlainColumn(price),
    }


def lineitem_q1(n: int, seed: int = 43, part=None, slicer=None):
    """Lineitem sorted by (returnflag, linestatus, shipdate, quantity):
    linestatus 'O' (1) iff shipdate > 1995-06-17, returnflag 'N' (1) for open
    lines else 'A' (0) / 'R' (2). Sorted key columns as runs (whole table, cut
    to this part's rows, snapped to quantity's runs); discount / tax / price
    positional."""
    rng = np.random.default_rng(seed)
    days = np.arange(SHIP_LO, SHIP_HI + 1, dtype=np.int64)
    dc = rng.multinomial(n, np.full(len(days), 1 / len(days)))
    open_ = days > 9298
    a_cnt = np.where(open_, 0, rng.binomial(dc, 0.5))
    groups = []  # (rf, ls, day, count) in sort order
    for rf in (0, 1, 2):
        for ls in (0, 1):
            if rf == 1:
                cnt = np.where(open_ if ls == 1 else np.zeros_like(open_), dc, 0)
            else:
                cnt = np.where(open_ | (ls == 1), 0, a_cnt if rf == 0 else dc - a_cnt)
            groups.append((rf, ls, cnt))
    rfv, rfc, lsv, lsc, shv, shc, qv, qc = [], [], [], [], [], [], [], []
    for rf, ls, cnt in groups:
        tot = int(cnt.sum())
        rfv.append([rf]); rfc.append([tot]); lsv.append([ls]); lsc.append([tot])
        shv.append(days); shc.append(cnt)
        for c in cnt[cnt > 0]:
            qv.append(np.arange(1, 51))
            qc.append(rng.multinomial(c, np.full(50, 1 / 50)))
    cat = lambda xs: np.concatenate([np.asarray(x) for x in xs])
    qty = _rle_from_counts(cat(qv), cat(qc), n)
    lo, hi = part_range(n, part, qty)
    # plain-centered i8 (storage = value − centre), the heuristic's pick for
    # these columns (tests/test_gpu_encode_choice.py)
    disc = positional(n, seed + 1, lo, hi, lambda r, m: (r.integers(0, 11, m) - DISC_CENTER).astype(np.int8), np.int8)
    tax = positional(n, seed + 2, lo, hi, lambda r, m: (r.integers(0, 9, m) - TAX_CENTER).astype(np.int8), np.int8)
    price = positional(n, seed + 3, lo, hi, lambda r, m: r.uniform(900.0, 105000.0, m), np.float64)
    return {
        "l_returnflag": cut(_rle_from_counts(cat(rfv), cat(rfc), n), lo, hi, slicer),
        "l_linestatus": cut(_rle_from_counts(cat(lsv), cat(lsc), n), lo, hi, slicer),
        "l_shipdate": cut(_rle_from_counts(cat(shv), cat(shc), n), lo, hi, slicer),
        "l_quantity": cut(qty, lo, hi, slicer),
        "l_discount": H.PlainColumn(disc, H.I64, DISC_CENTER),
        "l_tax": H.PlainColumn(tax, H.I64, TAX_CENTER),
        "l_extendedprice": H.PlainColumn(price),
    }


def q6(api, t) -> float:
    """SELECT SUM(l_extendedprice * l_discount) WHERE l_shipdate >= 1994-01-01
    AND l_shipdate < 1995-01-01 AND l_discount BETWEEN 5 AND 7 AND
    l_quantity < 24 — the acceptance Q6 plan shape (acceptance.cpp:399-415)."""
    C, M, A = api.compute, api.masks, api.agg
    m = M.and_mask(
        M.and_mask(C.compare_scalar(t["l_shipdate"], Q6_LO, ">="), C.compare_scalar(t["l_shipdate"], Q6_HI, "<")),
        M.and_mask(M.and_mask(C.compare_scalar(t["l_discount"], 5, ">="), C.compare_scalar(t["l_discount"], 7, "<=")),
                   C.compare_scalar(t["l_quantity"], 24, "<")))
    price = C.filter(t["l_extendedprice"], m)
    disc = C.filter(t["l_discount"], m)
    return A.aggregate_all(C.arith(price, disc, "*"), "sum")


Q1_FNS = ["sum", "sum", "sum", "sum", "avg", "avg", "avg", "count"]


# ---------------------------------------------------------------------------
# C5: production-shaped wide table
# ---------------------------------------------------------------------------

def _code_runs(n: int, avg: float, card: int, rng, dtype=np.int32) -> H.RleColumn:
    if avg >= n:
        return H.RleColumn(np.array([7], dtype), [0], [n - 1], n)
    e = run_ends(n, max(1, int(round(avg))), rng)
    s = np.concatenate([[0], e[:-1] + 1])
    return H.RleColumn(rng.integers(0, card, len(e)).astype(dtype), s, e, n)


def _plain_index(rng, n: int, frac: float = 0.01) -> H.PlainPlusIndexColumn:
    """i16 base (centre 0) + ~1% wide i64 outliers shadowing it (ingest.cpp
    plain_to_plain_index shape: base holds 0 at outlier rows)."""
    base = rng.integers(-30000, 30001, n).astype(np.int16)
    p = np.nonzero(rng.random(n) < frac)[0].astype(np.int64)
    base[p] = 0
    ov = rng.integers(-1_000_000_000, 1_000_000_001, len(p)).astype(np.int64)
    return H.PlainPlusIndexColumn(H.PlainColumn(base, H.I64, 0), H.IndexColumn(ov, p, n))


# C5 columns: RLE i32 dictionary codes (average run, cardinality), one single
# run, one with average run 34.41 (the paper's heaviest RLE column)
C5_RLE = {"r0": (None, 1), "r1": (34.41, 1000), "r2": (1e3, 100), "r3": (5e3, 100), "r4": (2e4, 50),
          "r5": (1e5, 20), "r6": (3e5, 10)}
# bit-width-reduced plain: (storage dtype, lo, hi, centre)
C5_PLAIN = {"p0": (np.int8, -100, 100, 1000), "p1": (np.int16, -20000, 20000, 50_000),
            "p2": (np.int32, -(1 << 30), (1 << 30) - 1, 0), "p3": (np.int16, -300, 300, None)}


def production_table(n: int, seed: int = 5, part=None, slicer=None, columns=None):
    """15 columns: 7 RLE i32 dictionary-code columns (one single run, one with
    average run 34.41 — the paper's heaviest RLE column, others 1e3..3e5),
    4 Plain+Index (i16 + 1% i64 outliers), 4 bit-width-reduced plain
    (i8 / i16 / i32 / i16 with centres). Every column has its own stream
    (RLE: whole table, cut to the part, cuts snapped to r2's runs; plain /
    Plain+Index: positional); `columns` limits what is generated."""
    names = columns or (list(C5_RLE) + [f"pi{i}" for i in range(4)] + list(C5_PLAIN))
    t = {}
    for i, c in enumerate(C5_RLE):
        if c in names or c == "r2":
            avg, card = C5_RLE[c]
            t[c] = _code_runs(n, n if avg is None else avg, card, np.random.default_rng([seed, 100 + i]))
    lo, hi = part_range(n, part, t["r2"])
    t = {c: cut(v, lo, hi, slicer) for c, v in t.items() if c in names}
    for i in range(4):
        if f"pi{i}" in names:
            t[f"pi{i}"] = positional_column(n, seed * 1000 + 10 + i, lo, hi, lambda r, m: _plain_index(r, m), slicer)
    for j, (c, (dt, a, b, centre)) in enumerate(C5_PLAIN.items()):
        if c in names:
            v = positional(n, seed * 1000 + 20 + j, lo, hi, lambda r, m, a=a, b=b, dt=dt: r.integers(a, b + 1, m).astype(dt),
                           dt)
            t[c] = H.PlainColumn(v, H.I64, centre)
    return t


C5_IN = (3, 17, 42)
C5_LT = 50
C5_FNS = ["sum", "sum", "count"]


def c5_query(api, t):
    """SELECT r4, SUM(pi0), SUM(p1), COUNT(*) WHERE r2 IN (3, 17, 42) AND
    r3 < 50 GROUP BY r4 — the production queries' semi-joins replaced by
    dictionary-code predicates (IN-list = OR of equalities)."""
    C, M, A = api.compute, api.masks, api.agg
    m_in = None
    for code in C5_IN:
        e = C.compare_scalar(t["r2"], code, "==")
        m_in = e if m_in is None else M.or_mask(m_in, e)
    m = M.and_mask(m_in, C.compare_scalar(t["r3"], C5_LT, "<"))
    f = {k: C.filter(t[k], m) for k in ("r4", "pi0", "p1")}
    return A.group_aggregate([f["r4"]], [f["pi0"], f["p1"], f["pi0"]], C5_FNS, normalize=True)


def q1(api, t):
    """SELECT rf, ls, SUM(qty), SUM(price), SUM(price*(100-disc)),
    SUM(price*(100-disc)*(100+tax)), AVG(qty), AVG(price), AVG(disc), COUNT(*)
    WHERE shipdate <= 1998-09-02 GROUP BY rf, ls (discount/tax in hundredths).
    Returns (keys, values, n_groups) as the group_aggregate call does."""
    C, A = api.compute, api.agg
    m = C.compare_scalar(t["l_shipdate"], Q1_CUTOFF, "<=")
    f = {k: C.filter(v, m) for k, v in t.items()}  # Filter applies to every scanned column
    disc_price = C.arith(f["l_extendedprice"], C.arith_scalar(f["l_discount"], 100, "-", True), "*")
    charge = C.arith(disc_price, C.arith_scalar(f["l_tax"], 100, "+"), "*")
    keys = [f["l_returnflag"], f["l_linestatus"]]
    data = [f["l_quantity"], f["l_extendedprice"], disc_price, charge, f["l_quantity"], f["l_extendedprice"],
            f["l_discount"], f["l_quantity"]]
    return A.group_aggregate(keys, data, Q1_FNS, normalize=True)


# ---------------------------------------------------------------------------
# Fused forms: the same plans through agg.group_aggregate_exprs (K12 — one
# pass over the compressed columns instead of materialised filter / arith
# outputs). `rq` is paper_2506_10092_b200.runq; the masks are built with the
# same compare_scalar / and_mask / or_mask calls as the chain plans above.
# ---------------------------------------------------------------------------


def q6_mask(api, t):
    C, M = api.compute, api.masks
    return M.and_mask(
        M.and_mask(C.compare_scalar(t["l_shipdate"], Q6_LO, ">="), C.compare_scalar(t["l_shipdate"], Q6_HI, "<")),
        M.and_mask(M.and_mask(C.compare_scalar(t["l_discount"], 5, ">="), C.compare_scalar(t["l_discount"], 7, "<=")),
                   C.compare_scalar(t["l_quantity"], 24, "<")))


Q6_WHERE = [("l_shipdate", ">=", Q6_LO), ("l_shipdate", "<", Q6_HI), ("l_discount", ">=", 5),
            ("l_discount", "<=", 7), ("l_quantity", "<", 24)]


def q6_prepared(rq, t, comm=None):
    """WHERE pushed into the fused call (conjuncts on RLE columns are
    evaluated per run segment; no mask is materialised), marshalled once:
    calling the result runs the query (agg.prepare_exprs). `comm`: this
    rank's shard, merged over the communicator."""
    X = rq.X
    plan = rq.agg.prepare_exprs(
        None, [], [X.col(t["l_extendedprice"]).arith(X.col(t["l_discount"]), "*")], ["sum"],
        where=[(t[c], op, k) for c, op, k in Q6_WHERE], comm=comm)

    def run():
        _, vs, _, fused = plan()
        v = vs[0]
        return (float(v.download()[0]) if hasattr(v, "download") else float(v[0])), fused
    return run


def q6_fused(rq, t, comm=None):
    return q6_prepared(rq, t, comm)()


def q1_prepared(rq, t, comm=None):
    X = rq.X
    price, disc, tax, qty = (t[k] for k in ("l_extendedprice", "l_discount", "l_tax", "l_quantity"))
    disc_price = X.col(price).arith(X.col(disc).scalar(100, "-", True), "*")
    charge = disc_price.arith(X.col(tax).scalar(100, "+"), "*")
    exprs = [X.col(qty), X.col(price), disc_price, charge, X.col(qty), X.col(price), X.col(disc), X.count()]
    plan = rq.agg.prepare_exprs(None, [t["l_returnflag"], t["l_linestatus"]], exprs, Q1_FNS,
                                where=[(t["l_shipdate"], "<=", Q1_CUTOFF)], comm=comm)

    def run():
        ks, vs, ng, fused = plan()
        return (ks, vs, ng), fused
    return run


def q1_fused(rq, t, comm=None):
    return q1_prepared(rq, t, comm)()


def c5_mask(api, t):
    C, M = api.compute, api.masks
    m_in = None
    for code in C5_IN:
        e = C.compare_scalar(t["r2"], code, "==")
        m_in = e if m_in is None else M.or_mask(m_in, e)
    return M.and_mask(m_in, C.compare_scalar(t["r3"], C5_LT, "<"))


def c5_prepared(rq, t, comm=None):
    X = rq.X
    plan = rq.agg.prepare_exprs(None, [t["r4"]], [X.col(t["pi0"]), X.col(t["p1"]), X.count()], C5_FNS,
                                where=[(t["r2"], "in", C5_IN), (t["r3"], "<", C5_LT)], comm=comm)

    def run():
        ks, vs, ng, fused = plan()
        return (ks, vs, ng), fused
    return run


def c5_fused(rq, t, comm=None):
    return c5_prepared(rq, t, comm)()
