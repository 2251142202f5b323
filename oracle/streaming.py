"""TEST INFRASTRUCTURE ONLY — the at-scale streaming oracle.

The reference cannot hold C3 at 10B rows (W alone is 80 GB) nor run it in
reasonable time (2.9M rows/s), so the group-by configurations C3, C4 Q1 /
Q6 and C5 are checked against this restatement instead, after it has been
pinned against the unmodified reference library on the same seeded tables
(tests/test_oracle_streaming_cpu.py; profiles/r2_oracle_validation.txt for
the 100M-row runs).

What it restates (reference file:line under proj/core):
  * runner.cpp:243-252 Filter applies the WHERE mask to every scanned
    column; runner.cpp:114-193 the mask is compare_scalar per literal
    (align.cpp:598-652, RLE branch: keep the passing runs), or_mask / and_mask
    of RLE masks (mask_ops.cpp:21-24 and_rle_rle = range_intersect);
  * runner.cpp:302-336 GroupAgg: normalize_basic, then group_aggregate
    (groupby.cpp:144-162: align_many → group_on_arrays → aggregate_array) or
    aggregate_all (groupby.cpp:164-172) when there are no keys;
  * groupby.cpp:67-135 aggregate_array: SUM int = Σ i64(v)·l wrapping, SUM
    float = Σ f64(v)·f64(l), COUNT = Σ l, AVG = f64(Σ v·l) / cnt;
  * kernels.cpp:154-186 unique_with_inverse: only groups that occur, keys
    ascending (lexicographic over the key columns).

The query becomes a segment table (row ranges of the key-run ∩ WHERE-run
intersection, one group slot each, orq_range_intersect in C) and every
aggregate input is folded over it by runq_oracle.c's orq_seg_sum_* (int64
wrapping sums, Neumaier f64 sums). Plain inputs fold in row chunks so a
table larger than host RAM streams through (`fold_plain_*` take row0).
Only tests/, __graft_entry__.smoke() and bench.py's gate / cpu_baseline /
reference legs import this module.
"""
from __future__ import annotations

import ctypes as C
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from paper_2506_10092_b200 import host as H

from .refpy import ORQ_SO, Orq

I64P = C.c_void_p


def _p(a: Optional[np.ndarray]):
    return C.c_void_p(a.ctypes.data if a is not None and a.size else None)


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64))


def _starts(col: H.RleColumn) -> np.ndarray:
    if col.s is not None:
        return _i64(col.s)
    return np.concatenate([[0], col.e[:-1] + 1]).astype(np.int64)


class Segments:
    """Disjoint ascending closed row ranges [ss, se] with a group slot each;
    `keys[k][g]` is key column k's value of slot g (slots ascending by key)."""

    def __init__(self, ss, se, slot, keys: List[np.ndarray], nslots: int):
        self.ss, self.se, self.slot = _i64(ss), _i64(se), _i64(slot)
        self.keys = keys
        self.nslots = nslots

    @property
    def n(self) -> int:
        return len(self.ss)


class StreamingOracle:
    def __init__(self):
        self.orq = Orq(ORQ_SO)
        L = self.orq.lib
        for name in ("orq_seg_sum_runs_i64", "orq_seg_sum_points_i64", "orq_seg_sum_plain_int",
                     "orq_seg_sum_plain_f64"):
            getattr(L, name).restype = None
        self.L = L

    # -- WHERE: RLE predicates → passing runs; conjunction by range_intersect --

    _CMP = {"<": np.less, "<=": np.less_equal, "==": np.equal, "!=": np.not_equal, ">=": np.greater_equal,
            ">": np.greater}

    def pred_runs(self, col: H.RleColumn, op: str, k) -> Tuple[np.ndarray, np.ndarray]:
        """compare_scalar RLE branch (align.cpp:598-652): the runs whose value
        passes, unmerged; an IN-list is the OR of equalities on one column
        (mask_ops.cpp or_mask of disjoint runs of the same column = the runs
        passing any of them, in order)."""
        v = np.asarray(col.v).astype(np.int64)
        ok = np.isin(v, np.asarray(k, np.int64)) if op == "in" else self._CMP[op](v, k)
        return _starts(col)[ok], _i64(col.e)[ok]

    def intersect(self, a, b):
        s, e, i1, i2 = self.orq.range_intersect(a[0], a[1], b[0], b[1])
        return (s, e), i1, i2

    def where_runs(self, preds: Sequence[Tuple[H.RleColumn, str, object]], total: int):
        runs = (np.array([0], np.int64), np.array([total - 1], np.int64))
        for col, op, k in preds:
            runs, _, _ = self.intersect(runs, self.pred_runs(col, op, k))
        return runs

    def segments(self, keys: Sequence[H.RleColumn], where=(), total: int = None) -> Segments:
        """Key runs ∩ WHERE runs; slot = rank of the key tuple among the tuples
        that occur (unique_with_inverse order, kernels.cpp:154-186)."""
        if total is None:
            total = (keys[0] if keys else where[0][0]).total_size
        runs = self.where_runs(where, total)
        key_vals = []
        for kc in keys:
            runs, i1, i2 = self.intersect(runs, (_starts(kc), _i64(kc.e)))
            key_vals = [kv[i1] for kv in key_vals] + [np.asarray(kc.v)[i2]]
        ss, se = runs
        if not keys:
            return Segments(ss, se, np.zeros(len(ss), np.int64), [], 1)
        order = np.lexsort(tuple(reversed([kv.astype(np.float64) if kv.dtype.kind == "f" else kv.astype(np.int64)
                                           for kv in key_vals])))
        cols = [kv[order] for kv in key_vals]
        brk = np.zeros(len(order), bool)
        if len(order):
            brk[0] = True
            for c in cols:
                brk[1:] |= c[1:] != c[:-1]
        gid = np.cumsum(brk) - 1
        slot = np.empty(len(order), np.int64)
        slot[order] = gid
        uniq = [c[brk] for c in cols]
        return Segments(ss, se, slot, uniq, int(brk.sum()))

    # -- folds ----------------------------------------------------------------

    def count(self, seg: Segments) -> np.ndarray:
        out = np.zeros(seg.nslots, np.int64)
        np.add.at(out, seg.slot, seg.se - seg.ss + 1)
        return out

    def fold_runs(self, seg: Segments, col: H.RleColumn, out=None, cnt=None) -> np.ndarray:
        out = np.zeros(seg.nslots, np.int64) if out is None else out
        v = _i64(col.v)
        s, e = _starts(col), _i64(col.e)
        self.L.orq_seg_sum_runs_i64(_p(seg.ss), _p(seg.se), _p(seg.slot), C.c_int64(seg.n), _p(v), _p(s), _p(e),
                                    C.c_int64(len(e)), _p(out), _p(cnt))
        return out

    def fold_points(self, seg: Segments, p, v, shadow: int = 0, out=None) -> np.ndarray:
        out = np.zeros(seg.nslots, np.int64) if out is None else out
        p, v = _i64(p), _i64(v)
        self.L.orq_seg_sum_points_i64(_p(seg.ss), _p(seg.se), _p(seg.slot), C.c_int64(seg.n), _p(p), _p(v),
                                      C.c_int64(len(p)), C.c_int64(shadow), _p(out), None)
        return out

    def fold_plain_int(self, seg: Segments, col: H.PlainColumn, row0: int = 0, out=None) -> np.ndarray:
        out = np.zeros(seg.nslots, np.int64) if out is None else out
        vals = np.ascontiguousarray(col.values)
        self.L.orq_seg_sum_plain_int(_p(seg.ss), _p(seg.se), _p(seg.slot), C.c_int64(seg.n),
                                     C.c_int64(seg.nslots), C.c_int64(row0), C.c_int64(len(vals)),
                                     C.c_int(H.dtype_code(vals)), _p(vals), C.c_int(col.logical),
                                     C.c_int(0 if col.center is None else 1), C.c_int64(col.center or 0), _p(out))
        return out

    def fold_plain_f64(self, seg: Segments, x: np.ndarray, row0: int = 0, seg_scale=None, f1=None, f2=None,
                       acc=None):
        """Σ x·f1·f2 per slot; f1/f2 = (narrow int array, mul, add) factors
        (double)(mul·d + add) per row, or seg_scale[i] per segment. `acc` is
        a (sum, comp) pair accumulated across chunks."""
        if acc is None:
            acc = (np.zeros(seg.nslots), np.zeros(seg.nslots))
        x = np.ascontiguousarray(x, np.float64)
        scale = None if seg_scale is None else np.ascontiguousarray(seg_scale, np.float64)

        def fac(f):
            if f is None:
                return (C.c_int(3), None, C.c_int64(0), C.c_int64(0), None)
            d = np.ascontiguousarray(f[0])
            return (C.c_int(H.dtype_code(d)), _p(d), C.c_int64(f[1]), C.c_int64(f[2]), d)

        a1, a2 = fac(f1), fac(f2)
        self.L.orq_seg_sum_plain_f64(_p(seg.ss), _p(seg.se), _p(seg.slot), C.c_int64(seg.n), C.c_int64(seg.nslots),
                                     C.c_int64(row0), C.c_int64(len(x)), _p(x), _p(scale), *a1[:4], *a2[:4],
                                     _p(acc[0]), _p(acc[1]))
        return acc


def f64_result(acc) -> np.ndarray:
    return acc[0] + acc[1]


def avg(sum_, cnt) -> np.ndarray:
    """AVG = f64 Σ / cnt, NaN for an empty group (groupby.cpp:103-106)."""
    cnt = np.asarray(cnt)
    with np.errstate(invalid="ignore", divide="ignore"):
        return np.where(cnt > 0, np.asarray(sum_, np.float64) / np.maximum(cnt, 1), np.nan)


def _present(seg: Segments, cnt: np.ndarray, keys_out, vals_out):
    """Drop slots no row reached (group_on_arrays only yields groups that
    occur): a WHERE can leave a key run with an empty intersection."""
    keep = cnt > 0
    return [k[keep] for k in keys_out], [v[keep] for v in vals_out]


# ---------------------------------------------------------------------------
# Partial tables: a configuration's oracle over ONE row range, in merge form
# (every column a SUM — int64 wrapping or f64 (sum, comp) — or a COUNT), so
# the oracle of a table cut into shards is merge(partials) → finish. The
# whole-table oracle is finish(partial(table)).
# ---------------------------------------------------------------------------


class Partial:
    def __init__(self, keys: List[np.ndarray], parts: list):
        self.keys, self.parts = keys, parts  # parts: int64 arrays or (sum, comp) f64 pairs


def merge(partials: Sequence[Partial]) -> Partial:
    """Union of the shards' groups, keys ascending; int64 parts wrap, f64
    parts add (Neumaier pairs kept)."""
    nk = len(partials[0].keys)
    if nk == 0:
        keys, inv, ng = [], [np.zeros(1, np.int64) for _ in partials], 1
    else:
        allk = [np.concatenate([p.keys[i].astype(np.float64 if p.keys[i].dtype.kind == "f" else np.int64)
                                for p in partials]) for i in range(nk)]
        order = np.lexsort(tuple(reversed(allk)))
        brk = np.zeros(len(order), bool)
        if len(order):
            brk[0] = True
            for k in allk:
                ks = k[order]
                brk[1:] |= ks[1:] != ks[:-1]
        gid = np.empty(len(order), np.int64)
        gid[order] = np.cumsum(brk) - 1
        ng = int(brk.sum())
        keys = [k[order][brk].astype(partials[0].keys[i].dtype) for i, k in enumerate(allk)]
        offs = np.cumsum([0] + [len(p.keys[0]) for p in partials])
        inv = [gid[offs[r]:offs[r + 1]] for r in range(len(partials))]
    parts = []
    for j, p0 in enumerate(partials[0].parts):
        if isinstance(p0, tuple):
            s, c = np.zeros(ng), np.zeros(ng)
            for r, p in enumerate(partials):
                np.add.at(s, inv[r], p.parts[j][0])
                np.add.at(c, inv[r], p.parts[j][1])
            parts.append((s, c))
        else:
            acc = np.zeros(ng, np.uint64)
            for r, p in enumerate(partials):
                np.add.at(acc, inv[r], p.parts[j].astype(np.int64).view(np.uint64))
            parts.append(acc.view(np.int64))
    return Partial(keys, parts)


def _val(x):
    return f64_result(x) if isinstance(x, tuple) else x


def _finish(p: Partial, spec):
    """spec: per output column, ("v", j) = part j as is, ("avg", j, c) =
    part j / part c; the count column of `cnt_at` drops empty groups."""
    cols = []
    for sp in spec:
        cols.append(_val(p.parts[sp[1]]) if sp[0] == "v" else avg(_val(p.parts[sp[1]]), p.parts[sp[2]]))
    return cols


# ---------------------------------------------------------------------------
# The configurations (each returns (keys, values) like group_aggregate)
# ---------------------------------------------------------------------------


class C3Fold:
    """C3: GROUP BY K → SUM(X), COUNT(*), AVG(Z), SUM(Y), SUM(W) over gapless
    columns (every row is in the joint alignment). RLE / RLE+Index inputs
    fold whole; the plain Z / W fold chunk by chunk via `add_plain_chunk`
    (row0 relative to the columns' first row)."""

    def __init__(self, so: StreamingOracle, k: H.RleColumn, x: H.RleColumn, y: H.RlePlusIndexColumn):
        self.so = so
        self.seg = so.segments([k])
        self.cnt = so.count(self.seg)
        self.sx = so.fold_runs(self.seg, x)
        self.sy = so.fold_runs(self.seg, y.runs)
        so.fold_points(self.seg, y.points.p, y.points.v, 0, out=self.sy)
        self.sz = np.zeros(self.seg.nslots, np.int64)
        self.sw = (np.zeros(self.seg.nslots), np.zeros(self.seg.nslots))

    def add_plain_chunk(self, row0: int, z: H.PlainColumn, w: np.ndarray):
        self.so.fold_plain_int(self.seg, z, row0, out=self.sz)
        self.so.fold_plain_f64(self.seg, w, row0, acc=self.sw)

    def partial(self) -> Partial:
        keys, parts = _present(self.seg, self.cnt, self.seg.keys, [self.sx, self.cnt, self.sz, self.sy])
        keep = self.cnt > 0
        return Partial(keys, parts + [(self.sw[0][keep], self.sw[1][keep])])

    def result(self):
        return c3_finish(self.partial())


def c3_finish(p: Partial):
    return p.keys, _finish(p, [("v", 0), ("v", 1), ("avg", 2, 1), ("v", 3), ("v", 4)])


def c3_partial(host: Dict[str, H.Column], so: StreamingOracle = None) -> Partial:
    so = so or StreamingOracle()
    f = C3Fold(so, host["k"], host["x"], host["y"])
    f.add_plain_chunk(0, host["z"], host["w"].values)
    return f.partial()


def c3(host: Dict[str, H.Column], so: StreamingOracle = None):
    return c3_finish(c3_partial(host, so))


def q1_partial(t: Dict[str, H.Column], cutoff: int, so: StreamingOracle = None) -> Partial:
    """Q1 (queries.q1): WHERE shipdate <= cutoff GROUP BY rf, ls → SUM(qty),
    SUM(price), SUM(price·(100−disc)), SUM(price·(100−disc)·(100+tax)),
    AVG(qty), AVG(price), AVG(disc), COUNT(*)."""
    so = so or StreamingOracle()
    seg = so.segments([t["l_returnflag"], t["l_linestatus"]], [(t["l_shipdate"], "<=", cutoff)])
    cnt = so.count(seg)
    sq = so.fold_runs(seg, t["l_quantity"])
    price = t["l_extendedprice"].values
    disc, tax = t["l_discount"], t["l_tax"]
    # decoded value = stored + centre (column.cpp:283-297): 100 − disc = −stored + (100 − centre)
    dc, tc = disc.center or 0, tax.center or 0
    sp = so.fold_plain_f64(seg, price)
    sdp = so.fold_plain_f64(seg, price, f1=(disc.values, -1, 100 - dc))
    sch = so.fold_plain_f64(seg, price, f1=(disc.values, -1, 100 - dc), f2=(tax.values, 1, 100 + tc))
    sd = so.fold_plain_int(seg, disc)
    keep = cnt > 0
    keys, ints = _present(seg, cnt, seg.keys, [sq, sd, cnt])
    f = [(a[0][keep], a[1][keep]) for a in (sp, sdp, sch)]
    return Partial(keys, ints + f)  # sq, sd, cnt, sp, sdp, sch


def q1_finish(p: Partial):
    return p.keys, _finish(p, [("v", 0), ("v", 3), ("v", 4), ("v", 5), ("avg", 0, 2), ("avg", 3, 2),
                               ("avg", 1, 2), ("v", 2)])


def q1(t: Dict[str, H.Column], cutoff: int, so: StreamingOracle = None):
    return q1_finish(q1_partial(t, cutoff, so))


def q6_partial(t: Dict[str, H.Column], where, so: StreamingOracle = None) -> Partial:
    """Q6: SUM(price·disc) under the five RLE conjuncts; disc is RLE in the
    Q6 sort order, so its value is constant over every segment (the
    segments include disc's runs)."""
    so = so or StreamingOracle()
    total = t["l_shipdate"].total_size
    seg = so.segments([t["l_discount"]], [(t[c], op, k) for c, op, k in where], total)
    # seg.keys[0][slot] is the discount of each segment
    scale = seg.keys[0][seg.slot].astype(np.float64)
    one = Segments(seg.ss, seg.se, np.zeros(seg.n, np.int64), [], 1)
    return Partial([], [so.fold_plain_f64(one, t["l_extendedprice"].values, seg_scale=scale)])


def q6_finish(p: Partial) -> float:
    return float(_val(p.parts[0])[0])


def q6(t: Dict[str, H.Column], where, so: StreamingOracle = None) -> float:
    return q6_finish(q6_partial(t, where, so))


def c5_partial(t: Dict[str, H.Column], in_list, lt: int, so: StreamingOracle = None) -> Partial:
    """C5: WHERE r2 IN (...) AND r3 < lt GROUP BY r4 → SUM(pi0), SUM(p1),
    COUNT(*); pi0 is Plain+Index (base folded as plain, outliers as points
    with the base's decode of 0 subtracted)."""
    so = so or StreamingOracle()
    seg = so.segments([t["r4"]], [(t["r2"], "in", in_list), (t["r3"], "<", lt)])
    cnt = so.count(seg)
    pi0 = t["pi0"]
    s0 = so.fold_plain_int(seg, pi0.base)
    shadow = int(np.int64(0) + np.int64(pi0.base.center or 0))
    so.fold_points(seg, pi0.outliers.p, pi0.outliers.v, shadow, out=s0)
    s1 = so.fold_plain_int(seg, t["p1"])
    keys, parts = _present(seg, cnt, seg.keys, [s0, s1, cnt])
    return Partial(keys, parts)


def c5_finish(p: Partial):
    return p.keys, _finish(p, [("v", 0), ("v", 1), ("v", 2)])


def c5(t: Dict[str, H.Column], in_list, lt: int, so: StreamingOracle = None):
    return c5_finish(c5_partial(t, in_list, lt, so))
