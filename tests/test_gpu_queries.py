"""GPU parity: TPC-H-style Q6 / Q1 (config C4) — the same plan functions run
through the device operator API and through the reference library."""
import numpy as np
import pytest

from helpers import assert_array, assert_scalar
from paper_2506_10092_b200 import queries as Q

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [1000, 250_000, 2_000_000])
def test_q6_device_vs_reference(rq, ref, n):
    from oracle.refpy import RefAPI
    t = Q.lineitem_q6(n, seed=n)
    assert_scalar(Q.q6(rq, t), Q.q6(RefAPI(ref), t), "q6")
    dt = {k: rq.upload(v) for k, v in t.items()}
    assert_scalar(Q.q6(rq, dt), Q.q6(RefAPI(ref), t), "q6 resident")


@pytest.mark.parametrize("n", [1000, 250_000])
def test_q1_device_vs_reference(rq, ref, n):
    from oracle.refpy import RefAPI
    t = Q.lineitem_q1(n, seed=n + 1)
    ks, vs, ng = Q.q1(rq, t)
    wk, wv, wng = Q.q1(RefAPI(ref), t)
    assert ng == wng
    for g, w in zip(ks + vs, wk + wv):
        assert_array(g, w)
