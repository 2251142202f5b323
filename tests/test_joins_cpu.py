"""CPU: pins the checker for joins::semi_join_mask — the reference library's
result against a row-level membership evaluation (test_join.cpp:194-214
shape: a probe row is set iff its value occurs in the build column)."""
import numpy as np
import pytest

from paper_2506_10092_b200 import datagen as G
from paper_2506_10092_b200 import host as H


def _rows(c):
    return H.column_rows(c)


def _bits(m, n):
    if isinstance(m, H.PlainMask):
        return m.bits.astype(bool)
    b = np.zeros(n, bool)
    if isinstance(m, H.RleMask):
        for s, e in zip(m.s, m.e):
            b[s:e + 1] = True
    elif isinstance(m, H.IndexMask):
        b[m.p] = True
    return b


@pytest.mark.parametrize("pe", [H.ENC_RLE, H.ENC_PLAIN, H.ENC_INDEX])
def test_reference_semi_join_matches_rows(ref, pe):
    rng = np.random.default_rng(151 + pe)
    for _ in range(20):
        n = 70
        probe = G.random_column(rng, pe, n, False, True, 6)
        build = G.random_column(rng, H.ENC_PLAIN, 30, False, True, 6)
        m = ref.semi_join_mask(probe, build)
        pos, vals = _rows(probe)
        bset = set(_rows(build)[1].tolist())
        want = np.zeros(n, bool)
        for p, v in zip(pos, vals):
            want[p] = v in bset
        assert np.array_equal(_bits(m, n), want)
