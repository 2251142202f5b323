"""GPU parity of joins::semi_join_mask (join.cpp:368-406) — the production
queries' semi-joins (§8f row 3) — against the reference library on the same
inputs: the reference's own test shape (test_join.cpp:194-214: RLE / Plain /
Index probes against a plain build), every encoding pair of the acceptance
combos (acceptance.cpp:300-330), float keys (−0 == +0; NaN by bit pattern),
composite inputs, empty sides and a million-run probe. Masks are compared
structurally: same encoding, same arrays."""
import numpy as np
import pytest

from helpers import assert_mask
from paper_2506_10092_b200 import datagen as G
from paper_2506_10092_b200 import host as H

pytestmark = pytest.mark.gpu
ENCS = [H.ENC_PLAIN, H.ENC_RLE, H.ENC_INDEX, H.ENC_PLAIN_INDEX, H.ENC_RLE_INDEX]


@pytest.mark.parametrize("pe", [H.ENC_RLE, H.ENC_PLAIN, H.ENC_INDEX])
def test_semi_join_reference_shape(rq, ref, pe):
    rng = np.random.default_rng(151 + pe)
    for it in range(20):
        probe = G.random_column(rng, pe, 70, False, True, 6)
        build = G.random_column(rng, H.ENC_PLAIN, 30, False, True, 6)
        assert_mask(rq.joins.semi_join_mask(probe, build), ref.semi_join_mask(probe, build), f"iter {it}")


@pytest.mark.parametrize("be", range(5))
@pytest.mark.parametrize("pe", range(5))
def test_semi_join_all_pairs(rq, ref, pe, be):
    rng = np.random.default_rng(1000 + 10 * pe + be)
    for it in range(5):
        n = int(rng.integers(1, 3000))
        probe = G.random_column(rng, ENCS[pe], n, bool(it % 2), True, 12)
        build = G.random_column(rng, ENCS[be], int(rng.integers(1, 2000)), bool(it % 3 == 0), True, 12)
        assert_mask(rq.joins.semi_join_mask(probe, build), ref.semi_join_mask(probe, build), f"iter {it}")


def test_semi_join_float_keys(rq, ref):
    probe = H.IndexColumn(np.array([0.0, -0.0, 1.5, np.nan, 2.0, 7.0]), np.arange(6, dtype=np.int64) * 3, 20)
    build = H.PlainColumn(np.array([-0.0, np.nan, 2, 9], dtype=np.float64))
    assert_mask(rq.joins.semi_join_mask(probe, build), ref.semi_join_mask(probe, build))
    ib = H.PlainColumn(np.array([2, 7, 0], dtype=np.int64))  # int build vs float probe: f64 domain
    assert_mask(rq.joins.semi_join_mask(probe, ib), ref.semi_join_mask(probe, ib))


def test_semi_join_empty_sides(rq, ref):
    probe = G.gapless_rle(1000, 10, 3, 0, 20)
    empty = H.IndexColumn(np.zeros(0, np.int64), np.zeros(0, np.int64), 50)
    assert_mask(rq.joins.semi_join_mask(probe, empty), ref.semi_join_mask(probe, empty))
    assert_mask(rq.joins.semi_join_mask(empty, probe), ref.semi_join_mask(empty, probe))


def test_semi_join_large_rle_probe(rq, ref):
    """A million-run dictionary-code column semi-joined with a 50K-key
    dimension: runs are probed, never expanded."""
    probe = G.gapless_rle(60_000_000, 60, 5, 0, 1_000_000)
    build = H.PlainColumn(np.random.default_rng(6).integers(0, 1_000_000, 50_000).astype(np.int64))
    got = rq.joins.semi_join_mask(rq.upload(probe), rq.upload(build)).download()
    assert_mask(got, ref.semi_join_mask(probe, build))
