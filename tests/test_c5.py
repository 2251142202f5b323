"""C5 production-shaped wide table: the plan (IN-list + '<' predicates,
GROUP BY an RLE code column) through the reference library vs a row-level
numpy evaluation (CPU), and through the device path vs the reference (GPU)."""
import numpy as np
import pytest

from helpers import assert_array
from paper_2506_10092_b200 import host as H
from paper_2506_10092_b200 import queries as Q


def rows(c):
    return H.column_rows(c)[1]


def test_c5_reference_plan_matches_sql(ref):
    from oracle.refpy import RefAPI
    t = Q.production_table(200_000, seed=9)
    ks, vs, ng = Q.c5_query(RefAPI(ref), t)
    r2, r3, r4, pi0, p1 = (rows(t[k]) for k in ("r2", "r3", "r4", "pi0", "p1"))
    sel = np.isin(r2, Q.C5_IN) & (r3 < Q.C5_LT)
    uk = np.unique(r4[sel])
    assert ng == len(uk) and np.array_equal(ks[0], uk)
    for i, key in enumerate(uk):
        g = sel & (r4 == key)
        assert vs[0][i] == int(pi0[g].astype(np.int64).sum())
        assert vs[1][i] == int(p1[g].astype(np.int64).sum())
        assert vs[2][i] == int(g.sum())


@pytest.mark.gpu
@pytest.mark.parametrize("n", [5_000, 400_000])
def test_c5_device_vs_reference(rq, ref, n):
    from oracle.refpy import RefAPI
    t = Q.production_table(n, seed=n)
    ks, vs, ng = Q.c5_query(rq, t)
    wk, wv, wng = Q.c5_query(RefAPI(ref), t)
    assert ng == wng
    for g, w in zip(ks + vs, wk + wv):
        assert_array(g, w)


@pytest.mark.gpu
def test_plain_index_filter_all_masks(rq, ref):
    """filter(Plain+Index, m) decodes only the selected rows — same result as
    the reference's decode-everything-then-gather for every mask encoding."""
    from paper_2506_10092_b200 import datagen as G
    rng = np.random.default_rng(4)
    for inst in range(6):
        n = int(rng.integers(10, 5000))
        c = G.random_column(rng, H.ENC_PLAIN_INDEX, n)
        for me in (H.MASK_PLAIN, H.MASK_RLE, H.MASK_INDEX, H.MASK_COMPOSITE):
            m = G.random_mask(rng, me, n)
            from helpers import assert_column
            assert_column(rq.compute.filter(c, m), ref.filter(c, m))
