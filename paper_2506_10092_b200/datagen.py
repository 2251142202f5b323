"""Seeded synthetic column generators (host numpy, no GPU).

* ``random_*`` restate the reference tests' generators
  (``proj/tests/oracle.hpp:122-256``: random_ranges / random_positions /
  random_mask / random_values / random_column) so the parity suites exercise
  the same shapes: gapped runs, sparse points, narrow plain + outliers,
  runs + points composites. (numpy's PCG64 replaces std::mt19937_64, so the
  instances differ; parity is always checked against the reference library
  on the SAME generated inputs.)
* ``gapless_rle`` / ``sparse_index`` / ``narrow_plain`` build the BASELINE
  config shapes: run lengths uniform in [1, 2L-1] tiling the
  domain, vectorised so 1B-10B-row tables generate in seconds.
"""
from __future__ import annotations

import numpy as np

from . import host as H


# ---------------------------------------------------------------------------
# reference-test-shaped generators (oracle.hpp:122-256)
# ---------------------------------------------------------------------------


def random_ranges(rng: np.random.Generator, n: int, density: float = 0.4):
    """Sorted, disjoint run list over [0, n) (oracle.hpp:122-137)."""
    s, e = [], []
    hi = max(1, n // 8)
    at = 0
    while at < n:
        ln = min(int(rng.integers(1, hi + 1)), n - at)
        if rng.random() < density:
            s.append(at)
            e.append(at + ln - 1)
        at += ln
    return np.array(s, dtype=np.int64), np.array(e, dtype=np.int64)


def random_positions(rng, n: int, density: float = 0.2):
    return np.nonzero(rng.random(n) < density)[0].astype(np.int64)


def random_values(rng, count: int, float_vals: bool, domain: int = 50):
    if float_vals:
        return rng.uniform(-100.0, 100.0, count)
    return rng.integers(-domain, domain + 1, count, dtype=np.int64)


def _covered(n, s, e):
    cov = np.zeros(n, dtype=bool)
    for a, b in zip(s, e):
        cov[a:b + 1] = True
    return cov


def random_mask(rng, enc: int, n: int):
    if enc == H.MASK_PLAIN:
        return H.PlainMask((rng.random(n) < 0.5).astype(np.uint8))
    if enc == H.MASK_RLE:
        s, e = random_ranges(rng, n)
        return H.RleMask(s, e, n)
    if enc == H.MASK_INDEX:
        return H.IndexMask(random_positions(rng, n), n)
    s, e = random_ranges(rng, n, 0.3)
    cov = _covered(n, s, e)
    pts = np.nonzero(~cov & (rng.random(n) < 0.15))[0]
    return H.CompositeMask(H.RleMask(s, e, n), H.IndexMask(pts, n))


def random_column(rng, enc: int, n: int, float_vals: bool = False, gaps: bool = True,
                  domain: int = 50):
    if enc == H.ENC_PLAIN:
        return H.PlainColumn(random_values(rng, n, float_vals, domain))
    if enc == H.ENC_RLE:
        s, e = random_ranges(rng, n, 0.5 if gaps else 1.0)
        return H.RleColumn(random_values(rng, len(s), float_vals, domain), s, e, n)
    if enc == H.ENC_INDEX:
        p = random_positions(rng, n, 0.25 if gaps else 1.0)
        return H.IndexColumn(random_values(rng, len(p), float_vals, domain), p, n)
    if enc == H.ENC_PLAIN_INDEX:
        # narrow int8 base plus sparse wide outliers (oracle.hpp:218-238)
        out = rng.random(n) < 0.05
        base = (rng.integers(-100, 101, n) // 2).astype(np.int8)
        base[out] = 0
        op = np.nonzero(out)[0].astype(np.int64)
        ov = rng.integers(1_000_000, 2_000_001, len(op), dtype=np.int64)
        return H.PlainPlusIndexColumn(H.PlainColumn(base, H.I64), H.IndexColumn(ov, op, n))
    s, e = random_ranges(rng, n, 0.35)
    runs = H.RleColumn(random_values(rng, len(s), float_vals, domain), s, e, n)
    cov = _covered(n, s, e)
    keep = ~cov & ((rng.random(n) < 0.2) if gaps else True)
    pp = np.nonzero(keep)[0].astype(np.int64)
    pts = H.IndexColumn(random_values(rng, len(pp), float_vals, domain), pp, n)
    return H.RlePlusIndexColumn(runs, pts)


# ---------------------------------------------------------------------------
# BASELINE config shapes
# ---------------------------------------------------------------------------


def run_ends(n: int, L: int, rng) -> np.ndarray:
    """End positions of runs with lengths uniform in [1, 2L-1] tiling [0, n)."""
    est = int(n / L * 1.02) + 64
    ends = []
    at = 0
    while at < n:
        lens = rng.integers(1, 2 * L, est, dtype=np.int64)
        e = at - 1 + np.cumsum(lens)
        cut = np.searchsorted(e, n - 1)
        if cut < len(e):
            e = e[:cut + 1]
            e[-1] = n - 1
            ends.append(e)
            break
        ends.append(e)
        at = int(e[-1]) + 1
    return np.concatenate(ends)


def gapless_rle(n: int, L: int, seed: int, lo: int = -1000, hi: int = 1000, dtype=np.int64) -> H.RleColumn:
    rng = np.random.default_rng(seed)
    e = run_ends(n, L, rng)
    s = np.empty_like(e)
    s[0] = 0
    s[1:] = e[:-1] + 1
    v = rng.integers(lo, hi + 1, len(e)).astype(dtype)
    return H.RleColumn(v, s, e, n)


def sparse_index(n: int, density: float, seed: int, lo: int = -1000, hi: int = 1000) -> H.IndexColumn:
    """Index column with ~density*n points (sorted unique positions)."""
    rng = np.random.default_rng(seed)
    k = int(n * density)
    # gaps between consecutive points ~ geometric(density): sorted, unique
    gaps = rng.geometric(density, k).astype(np.int64)
    p = np.cumsum(gaps) - 1
    p = p[p < n]
    v = rng.integers(lo, hi + 1, len(p)).astype(np.int64)
    return H.IndexColumn(v, p, n)


def narrow_plain(n: int, L: int, card: int, seed: int) -> H.PlainColumn:
    """Plain-centered i8 dictionary codes (ingest.cpp:261-266 shape): runs of
    length U[1, 2L-1] of codes in [0, card), stored as code - center."""
    rng = np.random.default_rng(seed)
    e = run_ends(n, L, rng)
    lens = np.diff(np.concatenate([[-1], e]))
    codes = rng.integers(0, card, len(e), dtype=np.int64)
    center = (card - 1) // 2
    vals = np.repeat((codes - center).astype(np.int8), lens)
    return H.PlainColumn(vals, H.I64, center)


def c1_tables(n: int = 10_000_000, la: int = 64, lb: int = 96, seed: int = 42):
    """C1: two misaligned gapless RLE int64 columns, values U[-1000, 1000]."""
    return gapless_rle(n, la, seed), gapless_rle(n, lb, seed + 1)


def c2_tables(n: int = 1_000_000_000, seed: int = 42, c_variant: str = "rle"):
    """C2: A RLE L=64, B Index 1%, C dictionary codes (cardinality 64):
    RLE L=256 (variant 'rle') or plain-centered i8 L=4 ('narrow')."""
    a = gapless_rle(n, 64, seed)
    b = sparse_index(n, 0.01, seed + 1)
    if c_variant == "rle":
        c = gapless_rle(n, 256, seed + 2, 0, 63)
    else:
        c = narrow_plain(n, 4, 64, seed + 2)
    return a, b, c


C2_K = 20  # C < 20 passes ~31% of rows


def rle_plus_index(n: int, L: int, point_frac: float, seed: int, lo: int = -1000,
                   hi: int = 1000) -> H.RlePlusIndexColumn:
    """RLE+Index covering every row: segments of length U[1, 2L-1]; a
    segment is expanded to single-row points with probability point_frac
    (so ~point_frac of the rows are points), else it is one run (the
    heuristic's 'rle+index' shape, ingest.cpp:217-271)."""
    rng = np.random.default_rng(seed)
    e = run_ends(n, L, rng)
    s = np.concatenate([[0], e[:-1] + 1])
    is_pt = rng.random(len(e)) < point_frac
    rs, re_ = s[~is_pt], e[~is_pt]
    rv = rng.integers(lo, hi + 1, len(rs)).astype(np.int64)
    ps, pe = s[is_pt], e[is_pt]
    lens = pe - ps + 1
    if len(lens):
        p = np.repeat(ps - np.concatenate([[0], np.cumsum(lens)[:-1]]), lens) + np.arange(lens.sum())
    else:
        p = np.empty(0, np.int64)
    pv = rng.integers(lo, hi + 1, len(p)).astype(np.int64)
    return H.RlePlusIndexColumn(H.RleColumn(rv, rs, re_, n), H.IndexColumn(pv, p.astype(np.int64), n))


C3_CHUNK = 1 << 28  # rows per generated chunk of C3's plain columns


def c3_run_columns(n: int, seed: int = 42):
    """C3's run-encoded columns: K codes 0..99 RLE L=4096, X RLE i64 L=128,
    Y RLE+Index (90% of rows in runs L=256, 10% points)."""
    k = gapless_rle(n, 4096, seed, 0, 99)
    x = gapless_rle(n, 128, seed + 1)
    y = rle_plus_index(n, 256, 0.1, seed + 2)
    return k, x, y


def c3_plain_chunk(n: int, seed: int, row0: int):
    """Rows [row0, row0 + C3_CHUNK) ∩ [0, n) of C3's plain columns: Z
    plain-centered i16 U[-20000, 20000] (logical i64) and W plain f64
    U[0, 100). Each chunk has its own stream, so a 10B-row table can be
    generated, uploaded and checked chunk by chunk."""
    assert row0 % C3_CHUNK == 0
    m = min(C3_CHUNK, n - row0)
    rng = np.random.default_rng([seed + 3, row0 // C3_CHUNK])
    z = rng.integers(-20000, 20001, m, dtype=np.int16)
    w = rng.uniform(0.0, 100.0, m)
    return z, w


def c3_tables(n: int, seed: int = 42):
    """C3: K, X, Y (c3_run_columns) + Z, W (c3_plain_chunk)."""
    k, x, y = c3_run_columns(n, seed)
    parts = [c3_plain_chunk(n, seed, r) for r in range(0, n, C3_CHUNK)]
    z = H.PlainColumn(np.concatenate([p[0] for p in parts]) if parts else np.empty(0, np.int16), H.I64, 0)
    w = H.PlainColumn(np.concatenate([p[1] for p in parts]) if parts else np.empty(0))
    return k, x, y, z, w


C3_FNS = ["sum", "count", "avg", "sum", "sum"]  # SUM(X), COUNT(*), AVG(Z), SUM(Y), SUM(W)
