"""CPU: the C4 plans (paper_2506_10092_b200.queries) run through the
reference library agree with a row-level numpy evaluation of the same SQL —
pins the plan restatement independently of both implementations."""
import numpy as np

from paper_2506_10092_b200 import host as H
from paper_2506_10092_b200 import queries as Q


def rows(c):
    return H.column_rows(c)[1]


def test_q6_reference_plan_matches_sql(ref):
    from oracle.refpy import RefAPI
    t = Q.lineitem_q6(300_000, seed=3)
    got = Q.q6(RefAPI(ref), t)
    sd, d, q, p = (rows(t[k]) for k in ("l_shipdate", "l_discount", "l_quantity", "l_extendedprice"))
    sel = (sd >= Q.Q6_LO) & (sd < Q.Q6_HI) & (d >= 5) & (d <= 7) & (q < 24)
    want = float(np.sum(p[sel] * d[sel]))
    assert abs(got - want) <= 1e-9 * max(1.0, abs(want))


def test_q1_reference_plan_matches_sql(ref):
    from oracle.refpy import RefAPI
    t = Q.lineitem_q1(300_000, seed=4)
    ks, vs, ng = Q.q1(RefAPI(ref), t)
    rf, ls, sd, q, d, tx, p = (rows(t[k]) for k in ("l_returnflag", "l_linestatus", "l_shipdate", "l_quantity",
                                                     "l_discount", "l_tax", "l_extendedprice"))
    sel = sd <= Q.Q1_CUTOFF
    g = rf[sel] * 2 + ls[sel]
    uk = np.unique(g)
    assert ng == len(uk)
    assert np.array_equal(ks[0], uk // 2) and np.array_equal(ks[1], uk % 2)
    dp = p[sel] * (100 - d[sel])
    ch = dp * (100 + tx[sel])
    cols = [q[sel], p[sel], dp, ch, q[sel], p[sel], d[sel], q[sel]]
    for v, col, fn in zip(vs, cols, Q.Q1_FNS):
        for i, key in enumerate(uk):
            x = col[g == key]
            want = {"sum": x.sum(), "avg": x.mean(), "count": len(x)}[fn]
            assert abs(float(v[i]) - float(want)) <= 1e-9 * max(1.0, abs(float(want))), (fn, i)
