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


def _assert_side(got, want, what):
    assert got[0] == want[0], f"{what}: side shape {got[0]} != {want[0]}"
    for g, w in zip(got[1:], want[1:]):
        assert np.array_equal(np.asarray(g, np.int64), np.asarray(w, np.int64)), f"{what}: {g} != {w}"


@pytest.mark.parametrize("re_", range(5))
@pytest.mark.parametrize("le", range(5))
def test_join_index_all_pairs(rq, ref, le, re_):
    """get_join_index in the reference's pairing order (acceptance.cpp:300-320
    combos), then apply_join_index of both sides onto columns of every
    encoding of those tables."""
    from helpers import assert_column
    rng = np.random.default_rng(3000 + 10 * le + re_)
    for it in range(3):
        nl, nr = int(rng.integers(1, 400)), int(rng.integers(1, 400))
        left = G.random_column(rng, ENCS[le], nl, False, True, 6)
        right = G.random_column(rng, ENCS[re_], nr, False, True, 6)
        gl, gr, gc = rq.joins.get_join_index(left, right)
        wl, wr, wc = ref.get_join_index(left, right)
        assert gc == wc, f"cardinality {gc} != {wc}"
        _assert_side(gl, wl, f"left iter {it}")
        _assert_side(gr, wr, f"right iter {it}")
        # apply each side to the table's columns (full-coverage encodings)
        for e2 in (H.ENC_PLAIN, H.ENC_RLE, H.ENC_INDEX, H.ENC_PLAIN_INDEX, H.ENC_RLE_INDEX):
            lc = G.random_column(rng, e2, nl, bool(it % 2), False, 20)
            rc = G.random_column(rng, e2, nr, bool(it % 2), False, 20)
            assert_column(rq.joins.apply_join_index(lc, wl), ref.apply_join_index(lc, wl), f"apply left enc {e2}")
            assert_column(rq.joins.apply_join_index(rc, wr), ref.apply_join_index(rc, wr), f"apply right enc {e2}")


def test_join_float_keys_and_many_to_many(rq, ref):
    left = H.RleColumn(np.array([1.0, -0.0, 2.5, 1.0]), np.array([0, 3, 5, 9], np.int64),
                       np.array([2, 4, 8, 11], np.int64), 12)
    right = H.RleColumn(np.array([0, 1, 1], np.int64), np.array([0, 2, 4], np.int64), np.array([1, 3, 6], np.int64), 7)
    gl, gr, gc = rq.joins.get_join_index(left, right)
    wl, wr, wc = ref.get_join_index(left, right)
    assert gc == wc
    _assert_side(gl, wl, "left")
    _assert_side(gr, wr, "right")


def test_apply_join_index_out_of_coverage_raises(rq):
    """test_join.cpp:189-193: a row reference outside the covered rows raises."""
    from paper_2506_10092_b200._lib import RqError
    gapped = H.RleColumn(np.array([1], np.int64), np.array([2], np.int64), np.array([4], np.int64), 10)
    with pytest.raises(RqError):
        rq.joins.apply_join_index(gapped, ("rows", np.array([0], np.int64)))
    with pytest.raises(RqError):
        rq.joins.apply_join_index(gapped, ("rle", np.array([0], np.int64), np.array([1], np.int64),
                                           np.array([3], np.int64)))


def test_hash_build_probe_vs_reference(rq, ref):
    rng = np.random.default_rng(71)
    for it in range(6):
        b = rng.integers(0, 40, int(rng.integers(0, 3000)))
        p = rng.integers(0, 40, int(rng.integers(0, 3000)))
        if it % 2:
            b = b.astype(np.float64)
        gb, gp = rq.joins.hash_build_probe(b, p)
        wb, wp = ref.hash_build_probe(b, p)
        assert np.array_equal(gb, wb) and np.array_equal(gp, wp), f"iter {it}"
