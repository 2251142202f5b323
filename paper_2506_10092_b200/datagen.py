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
    return _rle_plus_index_rng(np.random.default_rng(seed), n, L, point_frac, lo, hi)


def _rle_plus_index_rng(rng, n, L, point_frac, lo=-1000, hi=1000) -> H.RlePlusIndexColumn:
    e = run_ends(n, L, rng) if n > 0 else np.empty(0, np.int64)
    s = np.concatenate([[0], e[:-1] + 1]).astype(np.int64) if n > 0 else np.empty(0, np.int64)
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


# ---------------------------------------------------------------------------
# Row-range generation: a table of n rows is a deterministic function of its
# seed, and any row range [lo, hi) of it can be generated alone (one rank's
# shard of a table larger than any host, or a 10B-row column streamed into
# HBM chunk by chunk). Plain columns are positional: chunk c (rows
# [c·GEN_CHUNK, ...)) comes from its own stream default_rng([seed, c]).
# Run-encoded columns are either generated whole (few runs) and cut with a
# slicer (rq_shard_host_column on the device side, the numpy slicer in
# oracle/refpy on the checker side — the same function, tested equal), or
# chunk-positional too (runs end at chunk boundaries).
# ---------------------------------------------------------------------------

GEN_CHUNK = 50_000_000


def _chunks(n: int, lo: int, hi: int):
    for c in range(lo // GEN_CHUNK, (hi - 1) // GEN_CHUNK + 1) if hi > lo else ():
        r0 = c * GEN_CHUNK
        yield c, r0, min(GEN_CHUNK, n - r0)


def positional(n: int, seed: int, lo: int, hi: int, fn, dtype) -> np.ndarray:
    """Rows [lo, hi) of a plain column whose chunk c is fn(default_rng([seed, c]), rows)."""
    parts = []
    for c, r0, m in _chunks(n, lo, hi):
        a = fn(np.random.default_rng([seed, c]), m)
        parts.append(a[max(lo, r0) - r0:min(hi, r0 + m) - r0])
    return np.concatenate(parts).astype(dtype, copy=False) if parts else np.empty(0, dtype)


def _shift(col, off: int, total: int):
    if isinstance(col, H.RleColumn):
        return H.RleColumn(col.v, col.s + off, col.e + off, total)
    if isinstance(col, H.IndexColumn):
        return H.IndexColumn(col.v, col.p + off, total)
    if isinstance(col, H.RlePlusIndexColumn):
        return H.RlePlusIndexColumn(_shift(col.runs, off, total), _shift(col.points, off, total))
    if isinstance(col, H.PlainPlusIndexColumn):
        return H.PlainPlusIndexColumn(col.base, _shift(col.outliers, off, total))
    return col


def _concat(cols, total: int):
    c0 = cols[0]
    if isinstance(c0, H.RleColumn):
        return H.RleColumn(np.concatenate([c.v for c in cols]), np.concatenate([c.s for c in cols]),
                           np.concatenate([c.e for c in cols]), total)
    if isinstance(c0, H.IndexColumn):
        return H.IndexColumn(np.concatenate([c.v for c in cols]), np.concatenate([c.p for c in cols]), total)
    if isinstance(c0, H.RlePlusIndexColumn):
        return H.RlePlusIndexColumn(_concat([c.runs for c in cols], total), _concat([c.points for c in cols], total))
    if isinstance(c0, H.PlainPlusIndexColumn):
        base = H.PlainColumn(np.concatenate([c.base.values for c in cols]), c0.base.logical, c0.base.center)
        return H.PlainPlusIndexColumn(base, _concat([c.outliers for c in cols], total))
    return H.PlainColumn(np.concatenate([c.values for c in cols]), c0.logical, c0.center)


def positional_column(n: int, seed: int, lo: int, hi: int, fn, slicer=None):
    """Rows [lo, hi) of a column whose chunk c is the column fn(rng_c, rows)
    (runs / points end at chunk boundaries), positions rebased to lo."""
    chunks = list(_chunks(n, lo, hi))
    if not chunks:
        return fn(np.random.default_rng([seed, 0]), 0)
    span0 = chunks[0][1]
    span = chunks[-1][1] + chunks[-1][2] - span0
    col = _concat([_shift(fn(np.random.default_rng([seed, c]), m), r0 - span0, span) for c, r0, m in chunks], span)
    if (lo, hi) == (span0, span0 + span):
        return col
    assert slicer is not None, "a range not on chunk boundaries needs a slicer"
    return slicer(col, lo - span0, hi - span0)


def part_range(total: int, part, snap=None):
    """(lo, hi) of rank `part[0]` of `part[1]` (whole table when part is None),
    cut points snapped to `snap`'s run boundaries (sharding.plan_cuts)."""
    if part is None:
        return 0, total
    from .sharding import plan_cuts
    cuts = plan_cuts(total, part[1], snap)
    return cuts[part[0]], cuts[part[0] + 1]


def cut(col, lo: int, hi: int, slicer):
    if (lo, hi) == (0, col.total_size):
        return col
    return slicer(col, lo, hi)


def c3_run_columns(n: int, seed: int = 42, part=None, slicer=None):
    """C3's run-encoded columns over this part's rows: K codes 0..99 RLE
    L=4096, X RLE i64 L=128 (whole, cut; the cut points snap to X's runs),
    Y RLE+Index (90% of rows in runs L=256, 10% points; chunk-positional).
    Returns (k, x, y, lo, hi)."""
    k = gapless_rle(n, 4096, seed, 0, 99)
    x = gapless_rle(n, 128, seed + 1)
    lo, hi = part_range(n, part, x)
    y = positional_column(n, seed + 2, lo, hi, lambda rng, m: _rle_plus_index_rng(rng, m, 256, 0.1), slicer)
    return cut(k, lo, hi, slicer), cut(x, lo, hi, slicer), y, lo, hi


def c3_plain_rows(n: int, seed: int, lo: int, hi: int):
    """Rows [lo, hi) of C3's plain columns: Z plain-centered i16
    U[-20000, 20000] (logical i64) and W plain f64 U[0, 100)."""
    z = positional(n, seed + 3, lo, hi, lambda r, m: r.integers(-20000, 20001, m, dtype=np.int16), np.int16)
    w = positional(n, seed + 4, lo, hi, lambda r, m: r.uniform(0.0, 100.0, m), np.float64)
    return z, w


def c3_tables(n: int, seed: int = 42, part=None, slicer=None):
    """C3: K, X, Y, Z, W over this part's rows."""
    k, x, y, lo, hi = c3_run_columns(n, seed, part, slicer)
    z, w = c3_plain_rows(n, seed, lo, hi)
    return k, x, y, H.PlainColumn(z, H.I64, 0), H.PlainColumn(w)


C3_FNS = ["sum", "count", "avg", "sum", "sum"]  # SUM(X), COUNT(*), AVG(Z), SUM(Y), SUM(W)
