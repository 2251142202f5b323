"""Host-side column images mirroring the reference's column model.

The classes below restate ``runq::PlainColumn`` / ``RleColumn`` /
``IndexColumn`` / ``PlainPlusIndexColumn`` / ``RlePlusIndexColumn`` and the
four mask structs (``/root/reference/proj/core/include/runq/column.hpp:22-155``)
as numpy-backed dataclasses, plus their conversion to/from the flat C images
``rq_host_column`` / ``rq_host_mask`` declared in ``include/runq_b200.h``.

Pure host code: no device work happens here, so this module imports and
works without a GPU (the CPU test-suite uses it together with the oracle).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Union

import numpy as np

# runq::DType order (dtype.hpp:11)
I8, I16, I32, I64, F32, F64 = range(6)
DTYPES = {I8: np.int8, I16: np.int16, I32: np.int32, I64: np.int64, F32: np.float32, F64: np.float64}
DTYPE_NAMES = {I8: "i8", I16: "i16", I32: "i32", I64: "i64", F32: "f32", F64: "f64"}


def dtype_code(a) -> int:
    dt = np.dtype(a.dtype if hasattr(a, "dtype") else a)
    for code, npdt in DTYPES.items():
        if np.dtype(npdt) == dt:
            return code
    raise TypeError(f"unsupported dtype {dt}")


def is_float(code: int) -> bool:
    return code in (F32, F64)


# runq::Encoding / MaskEncoding (column.hpp:13-14)
ENC_PLAIN, ENC_RLE, ENC_INDEX, ENC_PLAIN_INDEX, ENC_RLE_INDEX = range(5)
MASK_PLAIN, MASK_RLE, MASK_INDEX, MASK_COMPOSITE = range(4)

# runq::compute::BinOp (align.hpp:70)
ADD, SUB, MUL, DIV, LT, LE, EQ, NE, GE, GT = range(10)
BINOP_NAMES = {"+": ADD, "-": SUB, "*": MUL, "/": DIV, "<": LT, "<=": LE, "==": EQ, "=": EQ,
               "!=": NE, "<>": NE, ">=": GE, ">": GT}
# runq::agg::AggFn (groupby.hpp:7)
SUM, COUNT, MIN, MAX, AVG, STD, VAR = range(7)
AGG_NAMES = {"sum": SUM, "count": COUNT, "min": MIN, "max": MAX, "avg": AVG, "std": STD, "var": VAR}


def _pos(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64))


def _vals(a, dtype=None) -> np.ndarray:
    if dtype is not None:
        return np.ascontiguousarray(np.asarray(a, dtype=dtype))
    a = np.asarray(a)
    if a.dtype == np.float64 or a.dtype == np.float32 or a.dtype in (np.int8, np.int16, np.int32, np.int64):
        return np.ascontiguousarray(a)
    if a.dtype.kind == "f":
        return np.ascontiguousarray(a.astype(np.float64))
    return np.ascontiguousarray(a.astype(np.int64))


# ---------------------------------------------------------------------------
# column images
# ---------------------------------------------------------------------------


@dataclass
class PlainColumn:
    """column.hpp:22-33 — values at storage width, logical type, optional centre."""
    values: np.ndarray
    logical: Optional[int] = None
    center: Optional[int] = None

    def __post_init__(self):
        self.values = _vals(self.values)
        if self.logical is None:
            self.logical = dtype_code(self.values)

    @property
    def total_size(self) -> int:
        return int(self.values.shape[0])

    encoding = ENC_PLAIN


@dataclass
class RleColumn:
    """column.hpp:38-49 — sorted disjoint closed runs [s_i, e_i] with values v."""
    v: np.ndarray
    s: np.ndarray
    e: np.ndarray
    total_size: int

    def __post_init__(self):
        self.v = _vals(self.v)
        # s may be None for a gapless column (runs tile [0, total_size)); the
        # C ABI then derives the starts on the device (runq_b200.h)
        self.s = _pos(self.s) if self.s is not None else None
        self.e = _pos(self.e)
        self.total_size = int(self.total_size)

    encoding = ENC_RLE

    def is_gapless(self) -> bool:
        if self.s is None:
            return True
        if len(self.e) == 0:
            return self.total_size == 0
        return bool(self.s[0] == 0 and self.e[-1] == self.total_size - 1 and np.array_equal(self.s[1:], self.e[:-1] + 1))

    def run_count(self) -> int:
        return int(self.s.shape[0])


@dataclass
class IndexColumn:
    """column.hpp:52-58 — sparse (value, position) pairs, strictly increasing p."""
    v: np.ndarray
    p: np.ndarray
    total_size: int

    def __post_init__(self):
        self.v = _vals(self.v)
        self.p = _pos(self.p)
        self.total_size = int(self.total_size)

    encoding = ENC_INDEX


@dataclass
class PlainPlusIndexColumn:
    """column.hpp:62-68 — narrow base + wide outliers shadowing the base."""
    base: PlainColumn
    outliers: IndexColumn

    encoding = ENC_PLAIN_INDEX

    @property
    def total_size(self) -> int:
        return self.base.total_size


@dataclass
class RlePlusIndexColumn:
    """column.hpp:71-76 — runs plus disjoint points."""
    runs: RleColumn
    points: IndexColumn

    encoding = ENC_RLE_INDEX

    @property
    def total_size(self) -> int:
        return self.runs.total_size


Column = Union[PlainColumn, RleColumn, IndexColumn, PlainPlusIndexColumn, RlePlusIndexColumn]


@dataclass
class PlainMask:
    bits: np.ndarray
    encoding = MASK_PLAIN

    def __post_init__(self):
        self.bits = np.ascontiguousarray(np.asarray(self.bits, dtype=np.uint8))

    @property
    def total_size(self) -> int:
        return int(self.bits.shape[0])


@dataclass
class RleMask:
    s: np.ndarray
    e: np.ndarray
    total_size: int
    encoding = MASK_RLE

    def __post_init__(self):
        self.s = _pos(self.s)
        self.e = _pos(self.e)
        self.total_size = int(self.total_size)


@dataclass
class IndexMask:
    p: np.ndarray
    total_size: int
    encoding = MASK_INDEX

    def __post_init__(self):
        self.p = _pos(self.p)
        self.total_size = int(self.total_size)


@dataclass
class CompositeMask:
    runs: RleMask
    points: IndexMask
    encoding = MASK_COMPOSITE

    @property
    def total_size(self) -> int:
        return self.runs.total_size


Mask = Union[PlainMask, RleMask, IndexMask, CompositeMask]


# ---------------------------------------------------------------------------
# C images (include/runq_b200.h)
# ---------------------------------------------------------------------------


class HostColumn(C.Structure):
    _fields_ = [
        ("encoding", C.c_int32), ("dtype", C.c_int32), ("logical", C.c_int32),
        ("has_center", C.c_int32), ("center", C.c_int64), ("total_size", C.c_int64),
        ("n", C.c_int64), ("v", C.c_void_p), ("s", C.c_void_p), ("e", C.c_void_p),
        ("p", C.c_void_p), ("dtype2", C.c_int32), ("_pad", C.c_int32), ("n2", C.c_int64),
        ("v2", C.c_void_p), ("p2", C.c_void_p),
    ]


class HostMask(C.Structure):
    _fields_ = [
        ("encoding", C.c_int32), ("_pad", C.c_int32), ("total_size", C.c_int64),
        ("n", C.c_int64), ("bits", C.c_void_p), ("s", C.c_void_p), ("e", C.c_void_p),
        ("p", C.c_void_p), ("n2", C.c_int64), ("p2", C.c_void_p),
    ]


class Scalar(C.Structure):
    _fields_ = [("is_float", C.c_int32), ("_pad", C.c_int32), ("i", C.c_int64), ("f", C.c_double)]


class Term(C.Structure):
    """rq_term: `col` (op = -1) or `col op k` / `k op col` (reversed)."""
    _fields_ = [("col", C.c_void_p), ("op", C.c_int32), ("reversed", C.c_int32), ("k", Scalar)]


class JoinSide(C.Structure):
    """rq_join_side: `rows` (is_rle = 0) or the ranges (v, s, e)."""
    _fields_ = [("is_rle", C.c_int32), ("_pad", C.c_int32), ("rows", C.c_void_p), ("v", C.c_void_p),
                ("s", C.c_void_p), ("e", C.c_void_p)]


class Pred(C.Structure):
    """rq_pred: `col op k`, or `col IN (in_list)` when n_in > 0."""
    _fields_ = [("col", C.c_void_p), ("op", C.c_int32), ("n_in", C.c_int32), ("k", Scalar),
                ("in_list", C.POINTER(Scalar))]


class Expr(C.Structure):
    """rq_expr: left-deep chain ((t0 ops[0] t1) ops[1] t2); n_terms 0 = COUNT(*)."""
    _fields_ = [("n_terms", C.c_int32), ("ops", C.c_int32 * 2), ("terms", Term * 3)]


# runq::io::Scheme (ingest.hpp:29)
SCHEME_PLAIN, SCHEME_PLAIN_CENTERED, SCHEME_RLE, SCHEME_RLE_INDEX, SCHEME_PLAIN_INDEX = range(5)
SCHEME_NAMES = {"plain": 0, "plain-centered": 1, "rle": 2, "rle+index": 3, "plain+index": 4}


class ColumnStats(C.Structure):
    """rq_column_stats = runq::ColumnStats (column.hpp:162-168)."""
    _fields_ = [("n_runs", C.c_int64), ("avg_run_length", C.c_double), ("encoded_bytes", C.c_int64),
                ("plain_bytes", C.c_int64), ("compression_ratio", C.c_double)]


class Heuristic(C.Structure):
    """runq::io::HeuristicConfig (ingest.hpp:41-48), reference defaults."""
    _fields_ = [("row_threshold", C.c_int64), ("ratio_threshold", C.c_double), ("trim", C.c_double),
                ("min_run", C.c_int64), ("unit_run_share", C.c_double)]

    def __init__(self, row_threshold=1_000_000, ratio_threshold=20.0, trim=0.05, min_run=2,
                 unit_run_share=0.5):
        super().__init__(row_threshold, ratio_threshold, trim, min_run, unit_run_share)


class EncodingChoice(C.Structure):
    """runq::io::EncodingChoice (ingest.hpp:33-39)."""
    _fields_ = [("scheme", C.c_int32), ("width", C.c_int32), ("min_run", C.c_int64),
                ("trim_fraction", C.c_double), ("has_center", C.c_int32), ("_pad", C.c_int32),
                ("center", C.c_int64)]

    def as_tuple(self):
        return (self.scheme, self.width, self.min_run, self.trim_fraction,
                self.center if self.has_center else None)


def make_scalar(k) -> Scalar:
    """runq::compute::Scalar = variant<int64_t, double> (align.hpp:76)."""
    if isinstance(k, (float, np.floating)):
        return Scalar(1, 0, 0, float(k))
    return Scalar(0, 0, int(k), 0.0)


def _ptr(a: Optional[np.ndarray]):
    if a is None or a.size == 0:
        return None
    return a.ctypes.data


def column_image(col: Column):
    """Returns (HostColumn, keepalive list)."""
    h = HostColumn()
    keep = []
    h.encoding = col.encoding
    h.total_size = col.total_size
    if isinstance(col, PlainColumn):
        h.dtype = dtype_code(col.values)
        h.logical = col.logical
        h.has_center = col.center is not None
        h.center = int(col.center or 0)
        h.n = col.values.shape[0]
        h.v = _ptr(col.values)
        keep.append(col.values)
    elif isinstance(col, RleColumn):
        h.dtype = h.logical = dtype_code(col.v)
        h.n = col.e.shape[0]
        h.v, h.s, h.e = _ptr(col.v), _ptr(col.s), _ptr(col.e)
        keep += [col.v, col.e] + ([col.s] if col.s is not None else [])
    elif isinstance(col, IndexColumn):
        h.dtype = h.logical = dtype_code(col.v)
        h.n = col.p.shape[0]
        h.v, h.p = _ptr(col.v), _ptr(col.p)
        keep += [col.v, col.p]
    elif isinstance(col, PlainPlusIndexColumn):
        b, o = col.base, col.outliers
        h.dtype = dtype_code(b.values)
        h.logical = b.logical
        h.has_center = b.center is not None
        h.center = int(b.center or 0)
        h.n = b.values.shape[0]
        h.v = _ptr(b.values)
        h.dtype2 = dtype_code(o.v)
        h.n2 = o.p.shape[0]
        h.v2, h.p2 = _ptr(o.v), _ptr(o.p)
        keep += [b.values, o.v, o.p]
    elif isinstance(col, RlePlusIndexColumn):
        r, q = col.runs, col.points
        h.dtype = h.logical = dtype_code(r.v)
        h.n = r.s.shape[0]
        h.v, h.s, h.e = _ptr(r.v), _ptr(r.s), _ptr(r.e)
        h.dtype2 = dtype_code(q.v)
        h.n2 = q.p.shape[0]
        h.v2, h.p2 = _ptr(q.v), _ptr(q.p)
        keep += [r.v, r.s, r.e, q.v, q.p]
    else:
        raise TypeError(f"not a column: {type(col)}")
    return h, keep


def alloc_for_image(h: HostColumn):
    """Allocates numpy arrays for a described image and points h at them."""
    arrs = {}
    enc = h.encoding
    n, n2 = int(h.n), int(h.n2)
    arrs["v"] = np.empty(n, dtype=DTYPES[h.dtype])
    if enc in (ENC_RLE, ENC_RLE_INDEX):
        arrs["s"] = np.empty(n, dtype=np.int64)
        arrs["e"] = np.empty(n, dtype=np.int64)
    if enc == ENC_INDEX:
        arrs["p"] = np.empty(n, dtype=np.int64)
    if enc in (ENC_PLAIN_INDEX, ENC_RLE_INDEX):
        arrs["v2"] = np.empty(n2, dtype=DTYPES[h.dtype2])
        arrs["p2"] = np.empty(n2, dtype=np.int64)
    for k, a in arrs.items():
        setattr(h, k, _ptr(a))
    return arrs


def column_from_image(h: HostColumn, arrs) -> Column:
    enc = h.encoding
    if enc == ENC_PLAIN:
        return PlainColumn(arrs["v"], int(h.logical), int(h.center) if h.has_center else None)
    if enc == ENC_RLE:
        return RleColumn(arrs["v"], arrs["s"], arrs["e"], int(h.total_size))
    if enc == ENC_INDEX:
        return IndexColumn(arrs["v"], arrs["p"], int(h.total_size))
    if enc == ENC_PLAIN_INDEX:
        base = PlainColumn(arrs["v"], int(h.logical), int(h.center) if h.has_center else None)
        return PlainPlusIndexColumn(base, IndexColumn(arrs["v2"], arrs["p2"], int(h.n)))
    if enc == ENC_RLE_INDEX:
        return RlePlusIndexColumn(RleColumn(arrs["v"], arrs["s"], arrs["e"], int(h.total_size)),
                                  IndexColumn(arrs["v2"], arrs["p2"], int(h.total_size)))
    raise ValueError(f"bad encoding {enc}")


def column_from_malloc_image(h: HostColumn) -> Column:
    """Copies a library-malloc'ed image (oracle shim / shard slicer) into numpy."""
    def take(ptr, n, dt):
        if n == 0 or not ptr:
            return np.empty(0, dtype=dt)
        buf = (C.c_char * (n * np.dtype(dt).itemsize)).from_address(ptr)
        return np.frombuffer(bytes(buf), dtype=dt).copy()
    n, n2 = int(h.n), int(h.n2)
    arrs = {"v": take(h.v, n, DTYPES[h.dtype])}
    if h.encoding in (ENC_RLE, ENC_RLE_INDEX):
        arrs["s"] = take(h.s, n, np.int64)
        arrs["e"] = take(h.e, n, np.int64)
    if h.encoding == ENC_INDEX:
        arrs["p"] = take(h.p, n, np.int64)
    if h.encoding in (ENC_PLAIN_INDEX, ENC_RLE_INDEX):
        arrs["v2"] = take(h.v2, n2, DTYPES[h.dtype2])
        arrs["p2"] = take(h.p2, n2, np.int64)
    return column_from_image(h, arrs)


def mask_image(m: Mask):
    h = HostMask()
    keep = []
    h.encoding = m.encoding
    h.total_size = m.total_size
    if isinstance(m, PlainMask):
        h.n = m.bits.shape[0]
        h.bits = _ptr(m.bits)
        keep.append(m.bits)
    elif isinstance(m, RleMask):
        h.n = m.s.shape[0]
        h.s, h.e = _ptr(m.s), _ptr(m.e)
        keep += [m.s, m.e]
    elif isinstance(m, IndexMask):
        h.n = m.p.shape[0]
        h.p = _ptr(m.p)
        keep.append(m.p)
    elif isinstance(m, CompositeMask):
        h.n = m.runs.s.shape[0]
        h.s, h.e = _ptr(m.runs.s), _ptr(m.runs.e)
        h.n2 = m.points.p.shape[0]
        h.p2 = _ptr(m.points.p)
        keep += [m.runs.s, m.runs.e, m.points.p]
    else:
        raise TypeError(f"not a mask: {type(m)}")
    return h, keep


def alloc_for_mask_image(h: HostMask):
    arrs = {}
    n, n2 = int(h.n), int(h.n2)
    if h.encoding == MASK_PLAIN:
        arrs["bits"] = np.empty(n, dtype=np.uint8)
    elif h.encoding == MASK_RLE:
        arrs["s"] = np.empty(n, dtype=np.int64)
        arrs["e"] = np.empty(n, dtype=np.int64)
    elif h.encoding == MASK_INDEX:
        arrs["p"] = np.empty(n, dtype=np.int64)
    else:
        arrs["s"] = np.empty(n, dtype=np.int64)
        arrs["e"] = np.empty(n, dtype=np.int64)
        arrs["p2"] = np.empty(n2, dtype=np.int64)
    for k, a in arrs.items():
        setattr(h, k, _ptr(a))
    return arrs


def mask_from_image(h: HostMask, arrs) -> Mask:
    t = int(h.total_size)
    if h.encoding == MASK_PLAIN:
        return PlainMask(arrs["bits"])
    if h.encoding == MASK_RLE:
        return RleMask(arrs["s"], arrs["e"], t)
    if h.encoding == MASK_INDEX:
        return IndexMask(arrs["p"], t)
    return CompositeMask(RleMask(arrs["s"], arrs["e"], t), IndexMask(arrs["p2"], t))


def mask_from_malloc_image(h: HostMask) -> Mask:
    def take(ptr, n, dt):
        if n == 0 or not ptr:
            return np.empty(0, dtype=dt)
        buf = (C.c_char * (n * np.dtype(dt).itemsize)).from_address(ptr)
        return np.frombuffer(bytes(buf), dtype=dt).copy()
    n, n2 = int(h.n), int(h.n2)
    arrs = {}
    if h.encoding == MASK_PLAIN:
        arrs["bits"] = take(h.bits, n, np.uint8)
    elif h.encoding == MASK_RLE:
        arrs["s"], arrs["e"] = take(h.s, n, np.int64), take(h.e, n, np.int64)
    elif h.encoding == MASK_INDEX:
        arrs["p"] = take(h.p, n, np.int64)
    else:
        arrs["s"], arrs["e"] = take(h.s, n, np.int64), take(h.e, n, np.int64)
        arrs["p2"] = take(h.p2, n2, np.int64)
    return mask_from_image(h, arrs)


# ---------------------------------------------------------------------------
# decoded views (the reference tests' oracle.hpp:20-95 decoders, restated)
# ---------------------------------------------------------------------------


def mask_bits(m: Mask) -> np.ndarray:
    """Byte-per-row bitmap of a mask's True set (oracle.hpp:20-48)."""
    out = np.zeros(m.total_size, dtype=np.uint8)
    if isinstance(m, PlainMask):
        out[:] = m.bits != 0
    elif isinstance(m, RleMask):
        _fill_runs(out, m.s, m.e)
    elif isinstance(m, IndexMask):
        out[m.p] = 1
    else:
        _fill_runs(out, m.runs.s, m.runs.e)
        out[m.points.p] = 1
    return out


def _fill_runs(out, s, e):
    if len(s) == 0:
        return
    d = np.zeros(out.shape[0] + 1, dtype=np.int64)
    np.add.at(d, s, 1)
    np.add.at(d, e + 1, -1)
    out[np.cumsum(d[:-1]) > 0] = 1


def decode_plain_values(c: PlainColumn) -> np.ndarray:
    """decode_values(PlainColumn) (column.cpp:283-297)."""
    logical = DTYPES[c.logical]
    if c.center is None and dtype_code(c.values) == c.logical:
        return c.values
    wide = c.values.astype(logical)
    if c.center is not None:
        wide = (wide.astype(np.int64) + np.int64(c.center)).astype(logical)
    return wide


def column_rows(c: Column):
    """(positions, values) over covered rows in row order (column.cpp:331-376)."""
    if isinstance(c, PlainColumn):
        return np.arange(c.total_size, dtype=np.int64), decode_plain_values(c)
    if isinstance(c, RleColumn):
        lens = c.e - c.s + 1
        if len(lens) == 0:
            return np.empty(0, np.int64), c.v[:0]
        pos = np.repeat(c.s - np.concatenate([[0], np.cumsum(lens)[:-1]]), lens) + np.arange(lens.sum())
        return pos.astype(np.int64), np.repeat(c.v, lens)
    if isinstance(c, IndexColumn):
        return c.p, c.v
    if isinstance(c, PlainPlusIndexColumn):
        vals = decode_plain_values(c.base).astype(DTYPES[dtype_code(c.outliers.v)])
        vals = vals.copy()
        vals[c.outliers.p] = c.outliers.v
        return np.arange(c.total_size, dtype=np.int64), vals
    rp, rv = column_rows(c.runs)
    pos = np.concatenate([rp, c.points.p])
    vals = np.concatenate([rv, c.points.v.astype(rv.dtype)])
    order = np.argsort(pos, kind="stable")
    return pos[order], vals[order]
