"""Python face of the B200 compressed-execution path, mirroring the
reference operator API (``runq::compute``, ``runq::enc``, ``runq::masks``,
``runq::agg``, ``runq::kernels``; align.hpp:59-95, primitives.hpp:28-92,
mask_ops.hpp:18, groupby.hpp:22-50, kernels.hpp:13-72) over the C ABI in
``include/runq_b200.h``.

Every function accepts host column images (``host.py``) or device handles.
Host inputs are uploaded and results downloaded (value semantics, like the
reference); device inputs stay resident and return device handles. All
compute runs in the sm_100a kernels of ``librunq_b200.so``; there is no
CPU fallback — the module raises at import if the library is missing.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Sequence, Tuple

import numpy as np

from . import host as H
from ._lib import RqDeviceError, RqError, RqOverflowError, RqResourceError, check, load  # noqa: F401

_L = load()


class Context:
    """rq_ctx_t: device, CUDA stream, stream-ordered pool, pinned readback."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(_L.rq_ctx_create(device, C.byref(h)))
        self.handle = h
        self.device = device

    def synchronize(self):
        check(_L.rq_ctx_synchronize(self.handle))

    @property
    def stream(self) -> int:
        return _L.rq_ctx_stream(self.handle) or 0

    @property
    def launches(self) -> int:
        return int(_L.rq_ctx_launches(self.handle))

    def close(self):
        if self.handle:
            _L.rq_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default = None


def default_context() -> Context:
    global _default
    if _default is None:
        _default = Context(0)
    return _default


def _ctx(ctx):
    return ctx if ctx is not None else default_context()


class DeviceArray:
    def __init__(self, handle, ctx: Context):
        self.handle = handle
        self.ctx = ctx

    @property
    def info(self):
        dt, n = C.c_int32(), C.c_int64()
        check(_L.rq_arr_info(self.handle, C.byref(dt), C.byref(n)))
        return int(dt.value), int(n.value)

    @property
    def dtype(self) -> int:
        return self.info[0]

    def __len__(self):
        return self.info[1]

    @property
    def device_ptr(self) -> int:
        return _L.rq_arr_device_ptr(self.handle) or 0

    def write(self, offset: int, host: np.ndarray):
        """rq_arr_write: host[...] → elements [offset, offset + len(host)).
        Stream-ordered: `host` must stay alive until the context syncs."""
        a = np.ascontiguousarray(host, dtype=H.DTYPES[self.dtype])
        check(_L.rq_arr_write(self.ctx.handle, self.handle, offset, a.ctypes.data if a.size else None,
                              a.shape[0]))
        return a

    def download(self) -> np.ndarray:
        dt, n = self.info
        out = np.empty(n, dtype=H.DTYPES[dt])
        check(_L.rq_arr_download(self.ctx.handle, self.handle, out.ctypes.data if n else None))
        return out

    def __del__(self):
        if getattr(self, "handle", None):
            _L.rq_arr_free(self.handle)
            self.handle = None


class DeviceColumn:
    """rq_col_t — a device-resident runq::Column."""

    def __init__(self, handle, ctx: Context):
        self.handle = handle
        self.ctx = ctx

    @property
    def encoding(self) -> int:
        return _L.rq_col_encoding(self.handle)

    @property
    def total_size(self) -> int:
        return int(_L.rq_col_total_size(self.handle))

    @property
    def value_type(self) -> int:
        return _L.rq_col_value_type(self.handle)

    def part(self, which: int) -> DeviceArray:
        h = C.c_void_p()
        check(_L.rq_col_part(self.handle, which, C.byref(h)))
        return DeviceArray(h, self.ctx)

    def download(self) -> H.Column:
        img = H.HostColumn()
        check(_L.rq_col_describe(self.handle, C.byref(img)))
        arrs = H.alloc_for_image(img)
        check(_L.rq_col_download(self.ctx.handle, self.handle, C.byref(img)))
        return H.column_from_image(img, arrs)

    def __del__(self):
        if getattr(self, "handle", None):
            _L.rq_col_free(self.handle)
            self.handle = None


class DeviceMask:
    """rq_mask_t — a device-resident runq::MaskColumn."""

    def __init__(self, handle, ctx: Context):
        self.handle = handle
        self.ctx = ctx

    def download(self) -> H.Mask:
        img = H.HostMask()
        check(_L.rq_mask_describe(self.handle, C.byref(img)))
        arrs = H.alloc_for_mask_image(img)
        check(_L.rq_mask_download(self.ctx.handle, self.handle, C.byref(img)))
        return H.mask_from_image(img, arrs)

    @property
    def encoding(self) -> int:
        img = H.HostMask()
        check(_L.rq_mask_describe(self.handle, C.byref(img)))
        return int(img.encoding)

    def true_count(self) -> int:
        n = C.c_int64()
        check(_L.rq_mask_true_count(self.ctx.handle, self.handle, C.byref(n)))
        return int(n.value)

    def __del__(self):
        if getattr(self, "handle", None):
            _L.rq_mask_free(self.handle)
            self.handle = None


def upload(x, ctx: Context = None):
    """Host column / mask / numpy array -> device handle."""
    ctx = _ctx(ctx)
    h = C.c_void_p()
    if isinstance(x, (DeviceColumn, DeviceMask, DeviceArray)):
        return x
    if isinstance(x, np.ndarray):
        a = np.ascontiguousarray(x)
        check(_L.rq_arr_upload(ctx.handle, H.dtype_code(a), a.ctypes.data if a.size else None,
                               a.shape[0], C.byref(h)))
        return DeviceArray(h, ctx)
    if isinstance(x, (H.PlainMask, H.RleMask, H.IndexMask, H.CompositeMask)):
        img, keep = H.mask_image(x)
        check(_L.rq_mask_upload(ctx.handle, C.byref(img), C.byref(h)))
        return DeviceMask(h, ctx)
    img, keep = H.column_image(x)
    check(_L.rq_col_upload(ctx.handle, C.byref(img), C.byref(h)))
    return DeviceColumn(h, ctx)


def alloc_array(dtype: int, n: int, ctx: Context = None) -> DeviceArray:
    """rq_arr_alloc: an uninitialised device array, filled by DeviceArray.write
    (columns larger than host RAM stream into HBM in row chunks)."""
    ctx = _ctx(ctx)
    h = C.c_void_p()
    check(_L.rq_arr_alloc(ctx.handle, dtype, n, C.byref(h)))
    return DeviceArray(h, ctx)


def make_plain(values: DeviceArray, logical: int = None, center=None) -> DeviceColumn:
    """rq_col_make_plain: a PlainColumn over a device array (shared)."""
    h = C.c_void_p()
    logical = values.dtype if logical is None else logical
    check(_L.rq_col_make_plain(values.ctx.handle, values.handle, logical, 0 if center is None else 1,
                               int(center or 0), C.byref(h)))
    return DeviceColumn(h, values.ctx)


def dump_image(col, ctx: Context = None) -> bytes:
    """rq_col_dump_image: the column's dump_column image (column.cpp:513-563)."""
    d = upload(col, ctx)
    p, n = C.c_void_p(), C.c_int64()
    check(_L.rq_col_dump_image(d.ctx.handle, d.handle, C.byref(p), C.byref(n)))
    try:
        return C.string_at(p, n.value)
    finally:
        _L.rq_image_free(p)


def load_image(image: bytes, ctx: Context = None) -> DeviceColumn:
    """rq_col_load_image: a dump_column image -> device column."""
    ctx = _ctx(ctx)
    h = C.c_void_p()
    buf = C.create_string_buffer(bytes(image), len(image))
    check(_L.rq_col_load_image(ctx.handle, buf, len(image), C.byref(h)))
    return DeviceColumn(h, ctx)


def _is_host(*xs) -> bool:
    return any(not isinstance(x, (DeviceColumn, DeviceMask, DeviceArray)) for x in xs)


def _out(dev, host_mode: bool):
    return dev.download() if host_mode else dev


def download_all(arrays):
    """Host copies of several device arrays (results of one query) with one
    synchronisation; host objects pass through unchanged."""
    dev = [a for a in arrays if isinstance(a, DeviceArray)]
    if not dev:
        return list(arrays)
    outs = {}
    for a in dev:
        dt, n = a.info
        outs[id(a)] = np.empty(n, dtype=H.DTYPES[dt])
    ctx = dev[0].ctx
    handles = (C.c_void_p * len(dev))(*[a.handle.value for a in dev])
    ptrs = (C.c_void_p * len(dev))(*[outs[id(a)].ctypes.data if outs[id(a)].size else None for a in dev])
    check(_L.rq_arr_download_many(ctx.handle, len(dev), handles, ptrs))
    return [outs[id(a)] if isinstance(a, DeviceArray) else a for a in arrays]


def _ctx_of(*xs) -> Context:
    for x in xs:
        if isinstance(x, (DeviceColumn, DeviceMask, DeviceArray)):
            return x.ctx
    return default_context()


def _new():
    return C.c_void_p()


def _arr_in(x, ctx, dtype=None):
    """numpy / list → device array (int64 unless the array has a dtype)."""
    if isinstance(x, DeviceArray):
        return x
    a = np.asarray(x) if dtype is None else np.asarray(x, dtype)
    if a.dtype == np.bool_:
        a = a.astype(np.int8)
    if dtype is None and a.dtype.kind in "iu" and a.dtype not in (np.int8, np.int16, np.int32, np.int64):
        a = a.astype(np.int64)
    return upload(np.ascontiguousarray(a), ctx)


def _arr_call(fn, ins, n_out, *scalars, dtype=np.int64, ctx=None):
    """Calls fn(ctx, *in_handles, *scalars, *out_ptrs) and returns the outputs
    (host arrays when any input was host, else device arrays)."""
    host = _is_host(*ins)
    ctx = ctx or _ctx_of(*ins)
    da = [_arr_in(x, ctx, dtype) for x in ins]
    outs = [_new() for _ in range(n_out)]
    check(fn(ctx.handle, *[a.handle for a in da], *scalars, *[C.byref(o) for o in outs]))
    res = tuple(_out(DeviceArray(o, ctx), host) if o.value else None for o in outs)
    return res[0] if n_out == 1 else res


class Shape:
    """compute::Shape (align.hpp:12-25): kind "dense" (n slots), "run" (s, e)
    or "point" (p)."""

    KINDS = ("dense", "run", "point")

    def __init__(self, kind, n=0, s=None, e=None, p=None):
        self.kind, self.n, self.s, self.e, self.p = kind, n, s, e, p

    @classmethod
    def _from(cls, kind, n, s, e, p, ctx, host):
        k = cls.KINDS[kind.value]
        get = lambda h: _out(DeviceArray(h, ctx), host) if h.value else None  # noqa: E731
        return cls(k, int(n.value), get(s), get(e), get(p))

    def _args(self, ctx):
        """ctypes arguments (kind, n, s, e, p); the uploaded arrays stay alive
        on the shape until the next call."""
        self._dev = [_arr_in(x, ctx, np.int64) if x is not None else None for x in (self.s, self.e, self.p)]
        return (C.c_int32(self.KINDS.index(self.kind)), C.c_int64(int(self.n if self.kind == "dense" else 0)),
                *[d.handle if d is not None else None for d in self._dev])

    def __repr__(self):
        return f"Shape({self.kind}, n={self.n})"


def _shape_outs():
    return C.c_int32(), C.c_int64(), _new(), _new(), _new()


# ---------------------------------------------------------------------------
# runq::enc (primitives.hpp:28-92) and runq::kernels (kernels.hpp:13-72)
# ---------------------------------------------------------------------------


class enc:
    @staticmethod
    def range_intersect(s1, e1, s2, e2):
        """enc::range_intersect (primitives.cpp:15-46) -> (s, e, idx1, idx2)."""
        host = _is_host(s1, e1, s2, e2)
        ctx = _ctx_of(s1, e1, s2, e2)
        a = [upload(np.asarray(x, np.int64) if not isinstance(x, DeviceArray) else x, ctx)
             for x in (s1, e1, s2, e2)]
        outs = [_new() for _ in range(4)]
        check(_L.rq_range_intersect(ctx.handle, *[x.handle for x in a], *[C.byref(o) for o in outs]))
        res = [DeviceArray(o, ctx) for o in outs]
        return tuple(_out(r, host) for r in res)

    @staticmethod
    def _points(fn, p, s, e):
        host = _is_host(p, s, e)
        ctx = _ctx_of(p, s, e)
        a = [upload(np.asarray(x, np.int64) if not isinstance(x, DeviceArray) else x, ctx)
             for x in (p, s, e)]
        outs = [_new() for _ in range(3)]
        check(fn(ctx.handle, *[x.handle for x in a], *[C.byref(o) for o in outs]))
        return tuple(_out(DeviceArray(o, ctx), host) for o in outs)

    @staticmethod
    def idx_in_rle(p, s, e):
        """enc::idx_in_rle (primitives.cpp:48-61) -> (p_out, run_of, idx_of)."""
        return enc._points(_L.rq_idx_in_rle, p, s, e)

    @staticmethod
    def rle_contain_idx(p, s, e):
        """enc::rle_contain_idx (primitives.cpp:63-86) -> (p_out, run_of, idx_of)."""
        return enc._points(_L.rq_rle_contain_idx, p, s, e)

    @staticmethod
    def idx_in_idx(p1, p2):
        """enc::idx_in_idx (primitives.cpp:88-100) -> (p_out, idx1, idx2)."""
        host = _is_host(p1, p2)
        ctx = _ctx_of(p1, p2)
        a = [upload(np.asarray(x, np.int64) if not isinstance(x, DeviceArray) else x, ctx)
             for x in (p1, p2)]
        outs = [_new() for _ in range(3)]
        check(_L.rq_idx_in_idx(ctx.handle, *[x.handle for x in a], *[C.byref(o) for o in outs]))
        return tuple(_out(DeviceArray(o, ctx), host) for o in outs)

    @staticmethod
    def plain_mask_to_rle(m):
        """enc::plain_mask_to_rle (primitives.cpp:349-360)."""
        host = _is_host(m)
        ctx = _ctx_of(m)
        dm = upload(m, ctx)
        o = _new()
        check(_L.rq_plain_mask_to_rle(ctx.handle, dm.handle, C.byref(o)))
        return _out(DeviceMask(o, ctx), host)

    @staticmethod
    def plain_mask_to_index(m):
        """enc::plain_mask_to_index (primitives.cpp:362-368)."""
        host = _is_host(m)
        ctx = _ctx_of(m)
        dm = upload(m, ctx)
        o = _new()
        check(_L.rq_plain_mask_to_index(ctx.handle, dm.handle, C.byref(o)))
        return _out(DeviceMask(o, ctx), host)

    @staticmethod
    def compact_rle(c):
        """enc::compact_rle (primitives.cpp:370-379)."""
        host = _is_host(c)
        ctx = _ctx_of(c)
        dc = upload(c, ctx)
        o = _new()
        check(_L.rq_compact_rle(ctx.handle, dc.handle, C.byref(o)))
        return _out(DeviceColumn(o, ctx), host)

    @staticmethod
    def plain_to_rle(c):
        """enc::plain_to_rle (primitives.cpp:223-250)."""
        host = _is_host(c)
        ctx = _ctx_of(c)
        dc = upload(c, ctx)
        o = _new()
        check(_L.rq_plain_to_rle(ctx.handle, dc.handle, C.byref(o)))
        return _out(DeviceColumn(o, ctx), host)

    @staticmethod
    def plain_to_rle_index(c, min_run: int):
        """enc::plain_to_rle_index (primitives.cpp:252-279)."""
        host = _is_host(c)
        ctx = _ctx_of(c)
        dc = upload(c, ctx)
        o = _new()
        check(_L.rq_plain_to_rle_index(ctx.handle, dc.handle, int(min_run), C.byref(o)))
        return _out(DeviceColumn(o, ctx), host)


    @staticmethod
    def plain_to_plain_index(c, trim_fraction: float):
        """enc::plain_to_plain_index (primitives.cpp:293-347)."""
        host = _is_host(c)
        ctx = _ctx_of(c)
        dc = upload(c, ctx)
        o = _new()
        check(_L.rq_plain_to_plain_index(ctx.handle, dc.handle, float(trim_fraction), C.byref(o)))
        return _out(DeviceColumn(o, ctx), host)

    @staticmethod
    def range_union(s1, e1, s2, e2):
        """enc::range_union (primitives.cpp:102-123) -> (s, e)."""
        return _arr_call(_L.rq_range_union, (s1, e1, s2, e2), 2)

    @staticmethod
    def merge_sorted_idx(p1, p2):
        """enc::merge_sorted_idx (primitives.cpp:125-131)."""
        return _arr_call(_L.rq_merge_sorted_idx, (p1, p2), 1)

    @staticmethod
    def concat_sort_idx(p1, p2):
        """enc::concat_sort_idx (primitives.cpp:133-139)."""
        return _arr_call(_L.rq_concat_sort_idx, (p1, p2), 1)

    @staticmethod
    def complement_rle(s, e, total: int):
        """enc::complement_rle (primitives.cpp:141-154) -> (s, e)."""
        host = _is_host(s, e)
        ctx = _ctx_of(s, e)
        a, b = _arr_in(s, ctx, np.int64), _arr_in(e, ctx, np.int64)
        so, eo = _new(), _new()
        check(_L.rq_complement_rle(ctx.handle, a.handle, b.handle, C.c_int64(total), C.byref(so), C.byref(eo)))
        return _out(DeviceArray(so, ctx), host), _out(DeviceArray(eo, ctx), host)

    @staticmethod
    def complement_index(p, total: int):
        """enc::complement_index (primitives.cpp:156-167) -> (s, e)."""
        host = _is_host(p)
        ctx = _ctx_of(p)
        a = _arr_in(p, ctx, np.int64)
        so, eo = _new(), _new()
        check(_L.rq_complement_index(ctx.handle, a.handle, C.c_int64(total), C.byref(so), C.byref(eo)))
        return _out(DeviceArray(so, ctx), host), _out(DeviceArray(eo, ctx), host)

    BUDGET = 1 << 33  # kDefaultElementBudget (primitives.hpp:12)

    @staticmethod
    def rle_to_index(c, budget: int = BUDGET):
        """enc::rle_to_index (primitives.cpp:172-192) for an RLE column or mask."""
        host = _is_host(c)
        ctx = _ctx_of(c)
        d = upload(c, ctx)
        o = _new()
        if isinstance(d, DeviceMask):
            check(_L.rq_mask_rle_to_index(ctx.handle, d.handle, C.c_int64(budget), C.byref(o)))
            return _out(DeviceMask(o, ctx), host)
        check(_L.rq_rle_to_index(ctx.handle, d.handle, C.c_int64(budget), C.byref(o)))
        return _out(DeviceColumn(o, ctx), host)

    @staticmethod
    def rle_to_plain(c, fill: float = 0.0, budget: int = BUDGET):
        """enc::rle_to_plain (primitives.cpp:194-218) for an RLE column or mask."""
        host = _is_host(c)
        ctx = _ctx_of(c)
        d = upload(c, ctx)
        o = _new()
        if isinstance(d, DeviceMask):
            check(_L.rq_mask_rle_to_plain(ctx.handle, d.handle, C.c_int64(budget), C.byref(o)))
            return _out(DeviceMask(o, ctx), host)
        check(_L.rq_rle_to_plain(ctx.handle, d.handle, C.c_double(fill), C.c_int64(budget), C.byref(o)))
        return _out(DeviceColumn(o, ctx), host)

    @staticmethod
    def compact_rle_index(c):
        """enc::compact_rle_index (primitives.cpp:381-420)."""
        host = _is_host(c)
        ctx = _ctx_of(c)
        d = upload(c, ctx)
        o = _new()
        check(_L.rq_compact_rle_index(ctx.handle, d.handle, C.byref(o)))
        return _out(DeviceColumn(o, ctx), host)


class io:
    """runq::io encoding selection and table sort (ingest.hpp:29-66), on the device."""
    Heuristic = H.Heuristic
    EncodingChoice = H.EncodingChoice

    @staticmethod
    def choose_encoding(c, cfg: "H.Heuristic" = None) -> "H.EncodingChoice":
        """io::choose_encoding (ingest.cpp:217-271)."""
        ctx = _ctx_of(c)
        dc = upload(c, ctx)
        out = H.EncodingChoice()
        check(_L.rq_choose_encoding(ctx.handle, dc.handle, C.byref(cfg) if cfg is not None else None,
                                    C.byref(out)))
        return out

    @staticmethod
    def encode(c, choice: "H.EncodingChoice"):
        """io::encode (ingest.cpp:273-290)."""
        host = _is_host(c)
        ctx = _ctx_of(c)
        dc = upload(c, ctx)
        o = _new()
        check(_L.rq_encode(ctx.handle, dc.handle, C.byref(choice), C.byref(o)))
        return _out(DeviceColumn(o, ctx), host)

    @staticmethod
    def sort_table(cols, by):
        """io::sort_table (ingest.cpp:292-344): cols is a list of plain
        columns (or a dict name -> column), by the key column indices (or names)."""
        names = None
        if isinstance(cols, dict):
            names = list(cols)
            by = [names.index(b) if isinstance(b, str) else b for b in by]
            cols = [cols[k] for k in names]
        host = _is_host(*cols)
        ctx = _ctx_of(*cols)
        dcs = [upload(c, ctx) for c in cols]
        handles = (C.c_void_p * len(dcs))(*[d.handle for d in dcs])
        bys = (C.c_int32 * len(by))(*by)
        outs = (C.c_void_p * len(dcs))()
        check(_L.rq_sort_table(ctx.handle, handles, len(dcs), bys, len(by), outs))
        res = [_out(DeviceColumn(C.c_void_p(h), ctx), host) for h in outs]
        return dict(zip(names, res)) if names is not None else res

    @staticmethod
    def encode_table(cols: dict, cfg: "H.Heuristic" = None) -> dict:
        """io::encode_table (ingest.cpp:346-357): choose + encode per column."""
        return {k: io.encode(c, io.choose_encoding(c, cfg)) for k, c in cols.items()}


class kernels:
    @staticmethod
    def bucketize(x, boundaries, right: bool):
        """kernels::bucketize (kernels.cpp:10-19)."""
        host = _is_host(x, boundaries)
        ctx = _ctx_of(x, boundaries)
        a = upload(np.asarray(x, np.int64) if not isinstance(x, DeviceArray) else x, ctx)
        b = upload(np.asarray(boundaries, np.int64) if not isinstance(boundaries, DeviceArray) else boundaries, ctx)
        o = _new()
        check(_L.rq_bucketize(ctx.handle, a.handle, b.handle, 1 if right else 0, C.byref(o)))
        return _out(DeviceArray(o, ctx), host)

    SUM, MIN, MAX, COUNT = range(4)  # kernels::Reduce (kernels.hpp:44)

    @staticmethod
    def cumsum(x, exclusive: bool):
        """kernels::cumsum (kernels.cpp:21-31); int64 overflow raises RqOverflowError."""
        return _arr_call(_L.rq_cumsum, (x,), 1, C.c_int32(1 if exclusive else 0))

    @staticmethod
    def checked_sum(x) -> int:
        """kernels::checked_sum (kernels.cpp:33-38)."""
        ctx = _ctx_of(x)
        a = _arr_in(x, ctx, np.int64)
        out = C.c_int64()
        check(_L.rq_checked_sum(ctx.handle, a.handle, C.byref(out)))
        return int(out.value)

    @staticmethod
    def repeat_interleave(values, counts):
        """kernels::repeat_interleave (kernels.cpp:40-45)."""
        host = _is_host(values, counts)
        ctx = _ctx_of(values, counts)
        v, c = _arr_in(values, ctx), _arr_in(counts, ctx, np.int64)
        o = _new()
        check(_L.rq_repeat_interleave(ctx.handle, v.handle, c.handle, C.byref(o)))
        return _out(DeviceArray(o, ctx), host)

    @staticmethod
    def range_arange(start, length):
        """kernels::range_arange (kernels.cpp:47-60)."""
        return _arr_call(_L.rq_range_arange, (start, length), 1)

    @staticmethod
    def scatter_reduce(values, index, n_groups: int, op):
        """kernels::scatter_reduce (kernels.cpp:97-125); op = kernels.SUM/MIN/MAX/COUNT
        or its name."""
        op = {"sum": 0, "min": 1, "max": 2, "count": 3}.get(op, op)
        host = _is_host(values, index)
        ctx = _ctx_of(values, index)
        v, i = _arr_in(values, ctx), _arr_in(index, ctx, np.int64)
        o = _new()
        check(_L.rq_scatter_reduce(ctx.handle, v.handle, i.handle, C.c_int64(n_groups), C.c_int32(op), C.byref(o)))
        return _out(DeviceArray(o, ctx), host)

    @staticmethod
    def unique_with_inverse(columns):
        """kernels::unique_with_inverse (kernels.cpp:127-187) -> (keys, inverse, n_groups)."""
        host = _is_host(*columns)
        ctx = _ctx_of(*columns)
        ds = [_arr_in(c, ctx) for c in columns]
        arr = (C.c_void_p * max(1, len(ds)))(*[d.handle.value for d in ds])
        ko = (C.c_void_p * max(1, len(ds)))()
        inv, ng = _new(), C.c_int64()
        check(_L.rq_unique_with_inverse(ctx.handle, arr, len(ds), ko, C.byref(inv), C.byref(ng)))
        keys = [_out(DeviceArray(C.c_void_p(ko[i]), ctx), host) for i in range(len(ds))]
        return keys, _out(DeviceArray(inv, ctx), host), int(ng.value)

    @staticmethod
    def gather(values, idx):
        """kernels::gather (kernels.cpp:195-219); out-of-range raises RqError."""
        host = _is_host(values, idx)
        ctx = _ctx_of(values, idx)
        v, i = _arr_in(values, ctx), _arr_in(idx, ctx, np.int64)
        o = _new()
        check(_L.rq_gather(ctx.handle, v.handle, i.handle, C.byref(o)))
        return _out(DeviceArray(o, ctx), host)

    @staticmethod
    def sort_with_perm(values):
        """kernels::sort_with_perm (kernels.cpp:221-233) -> (sorted, perm)."""
        host = _is_host(values)
        ctx = _ctx_of(values)
        v = _arr_in(values, ctx)
        so, pe = _new(), _new()
        check(_L.rq_sort_with_perm(ctx.handle, v.handle, C.byref(so), C.byref(pe)))
        return _out(DeviceArray(so, ctx), host), _out(DeviceArray(pe, ctx), host)

    @staticmethod
    def adjacent_ne(x):
        """kernels::adjacent_ne (kernels.cpp:235-245) -> uint8 0/1."""
        host = _is_host(x)
        ctx = _ctx_of(x)
        v = _arr_in(x, ctx)
        o = _new()
        check(_L.rq_adjacent_ne(ctx.handle, v.handle, C.byref(o)))
        r = _out(DeviceArray(o, ctx), host)
        return r.view(np.uint8) if host else r


# ---------------------------------------------------------------------------
# column model helpers
# ---------------------------------------------------------------------------


def decode_values(c):
    """decode_values (column.cpp:283-309) for Plain / Plain+Index."""
    host = _is_host(c)
    ctx = _ctx_of(c)
    dc = upload(c, ctx)
    o = _new()
    check(_L.rq_decode_values(ctx.handle, dc.handle, C.byref(o)))
    return _out(DeviceArray(o, ctx), host)


def _host_arr(x):
    return x.download() if isinstance(x, DeviceArray) else np.asarray(x)


def decode_full(c):
    """decode_full (column.cpp:311-329): values of a gap-free column (gaps raise RqError)."""
    host = _is_host(c)
    ctx = _ctx_of(c)
    dc = upload(c, ctx)
    o = _new()
    check(_L.rq_decode_full(ctx.handle, dc.handle, C.byref(o)))
    return _out(DeviceArray(o, ctx), host)


def to_rows(c):
    """to_rows (column.cpp:331-376) -> (positions, values) of the covered rows."""
    host = _is_host(c)
    ctx = _ctx_of(c)
    dc = upload(c, ctx)
    p, v = _new(), _new()
    check(_L.rq_to_rows(ctx.handle, dc.handle, C.byref(p), C.byref(v)))
    return _out(DeviceArray(p, ctx), host), _out(DeviceArray(v, ctx), host)


def stats(c) -> dict:
    """stats (column.cpp:244-279): the reference's byte accounting."""
    ctx = _ctx_of(c)
    dc = upload(c, ctx)
    st = H.ColumnStats()
    check(_L.rq_col_stats(ctx.handle, dc.handle, C.byref(st)))
    return {"n_runs": st.n_runs, "avg_run_length": st.avg_run_length, "encoded_bytes": st.encoded_bytes,
            "plain_bytes": st.plain_bytes, "compression_ratio": st.compression_ratio}


# ---------------------------------------------------------------------------
# runq::compute (align.hpp:59-95)
# ---------------------------------------------------------------------------


class compute:
    DENSE, RUN, POINT = 0, 1, 2
    Shape = Shape

    @staticmethod
    def decompose(c):
        """compute::decompose (align.cpp:86-100) -> (Shape, values)."""
        host = _is_host(c)
        ctx = _ctx_of(c)
        dc = upload(c, ctx)
        k, n, ps, pe, pp = _shape_outs()
        v = _new()
        check(_L.rq_decompose(ctx.handle, dc.handle, C.byref(k), C.byref(n), C.byref(ps), C.byref(pe), C.byref(pp),
                              C.byref(v)))
        return Shape._from(k, n, ps, pe, pp, ctx, host), _out(DeviceArray(v, ctx), host)

    @staticmethod
    def align_many(cols):
        """compute::align_many (align.cpp:233-254) -> (Shape, [values per column])."""
        host = _is_host(*cols)
        ctx = _ctx_of(*cols)
        dcs = [upload(c, ctx) for c in cols]
        arr = (C.c_void_p * len(dcs))(*[d.handle.value for d in dcs])
        vals = (C.c_void_p * len(dcs))()
        k, n, ps, pe, pp = _shape_outs()
        check(_L.rq_align_many(ctx.handle, arr, len(dcs), C.byref(k), C.byref(n), C.byref(ps), C.byref(pe),
                               C.byref(pp), vals))
        return (Shape._from(k, n, ps, pe, pp, ctx, host),
                [_out(DeviceArray(C.c_void_p(vals[i]), ctx), host) for i in range(len(dcs))])

    @staticmethod
    def shape_weights(sh: Shape):
        """compute::shape_weights (align.cpp:57-70)."""
        ins = [x for x in (sh.s, sh.e, sh.p) if x is not None]
        host = _is_host(*ins) if ins else True
        ctx = _ctx_of(*ins)
        o = _new()
        check(_L.rq_shape_weights(ctx.handle, *sh._args(ctx), C.byref(o)))
        return _out(DeviceArray(o, ctx), host)

    @staticmethod
    def normalize_basic(c):
        """compute::normalize_basic (align.cpp:102-115)."""
        host = _is_host(c)
        ctx = _ctx_of(c)
        dc = upload(c, ctx)
        o = _new()
        check(_L.rq_normalize_basic(ctx.handle, dc.handle, C.byref(o)))
        return _out(DeviceColumn(o, ctx), host)

    @staticmethod
    def align(a, b):
        """compute::align (align.cpp:219-231) -> dict(kind, s, e, p, v1, v2, total_size)."""
        host = _is_host(a, b)
        ctx = _ctx_of(a, b)
        da, db = upload(a, ctx), upload(b, ctx)
        kind = C.c_int32()
        outs = [_new() for _ in range(5)]
        check(_L.rq_align(ctx.handle, da.handle, db.handle, C.byref(kind), *[C.byref(o) for o in outs]))
        res = {"kind": int(kind.value), "total_size": da.total_size}
        for name, o in zip(("s", "e", "p", "v1", "v2"), outs):
            res[name] = _out(DeviceArray(o, ctx), host) if o.value else None
        return res

    @staticmethod
    def arith(a, b, op):
        """compute::arith (align.cpp:495-508)."""
        op = H.BINOP_NAMES.get(op, op)
        host = _is_host(a, b)
        ctx = _ctx_of(a, b)
        da, db = upload(a, ctx), upload(b, ctx)
        o = _new()
        check(_L.rq_arith(ctx.handle, da.handle, db.handle, op, C.byref(o)))
        return _out(DeviceColumn(o, ctx), host)

    @staticmethod
    def compare(a, b, op):
        """compute::compare (align.cpp:510-523)."""
        op = H.BINOP_NAMES.get(op, op)
        host = _is_host(a, b)
        ctx = _ctx_of(a, b)
        da, db = upload(a, ctx), upload(b, ctx)
        o = _new()
        check(_L.rq_compare(ctx.handle, da.handle, db.handle, op, C.byref(o)))
        return _out(DeviceMask(o, ctx), host)

    @staticmethod
    def binary_op(a, b, op):
        """compute::binary_op (align.cpp:525-528)."""
        op = H.BINOP_NAMES.get(op, op)
        return compute.compare(a, b, op) if op >= H.LT else compute.arith(a, b, op)

    @staticmethod
    def arith_scalar(a, k, op, reversed: bool = False):
        """compute::arith_scalar (align.cpp:571-596)."""
        op = H.BINOP_NAMES.get(op, op)
        host = _is_host(a)
        ctx = _ctx_of(a)
        da = upload(a, ctx)
        o = _new()
        check(_L.rq_arith_scalar(ctx.handle, da.handle, H.make_scalar(k), op, 1 if reversed else 0, C.byref(o)))
        return _out(DeviceColumn(o, ctx), host)

    @staticmethod
    def compare_scalar(a, k, op, reversed: bool = False):
        """compute::compare_scalar (align.cpp:598-652)."""
        op = H.BINOP_NAMES.get(op, op)
        host = _is_host(a)
        ctx = _ctx_of(a)
        da = upload(a, ctx)
        o = _new()
        check(_L.rq_compare_scalar(ctx.handle, da.handle, H.make_scalar(k), op, 1 if reversed else 0, C.byref(o)))
        return _out(DeviceMask(o, ctx), host)

    @staticmethod
    def scalar_op(a, k, op, reversed: bool = False):
        """compute::scalar_op (align.cpp:654-657)."""
        op = H.BINOP_NAMES.get(op, op)
        if op >= H.LT:
            return compute.compare_scalar(a, k, op, reversed)
        return compute.arith_scalar(a, k, op, reversed)

    @staticmethod
    def filter(a, m):
        """compute::filter (align.cpp:755-771)."""
        host = _is_host(a, m)
        ctx = _ctx_of(a, m)
        da, dm = upload(a, ctx), upload(m, ctx)
        o = _new()
        check(_L.rq_filter(ctx.handle, da.handle, dm.handle, C.byref(o)))
        return _out(DeviceColumn(o, ctx), host)


class masks:
    @staticmethod
    def and_mask(a, b):
        """masks::and_mask (mask_ops.cpp:183-209)."""
        host = _is_host(a, b)
        ctx = _ctx_of(a, b)
        da, db = upload(a, ctx), upload(b, ctx)
        o = _new()
        check(_L.rq_mask_and(ctx.handle, da.handle, db.handle, C.byref(o)))
        return _out(DeviceMask(o, ctx), host)

    @staticmethod
    def or_mask(a, b):
        """masks::or_mask (mask_ops.cpp:211-237)."""
        host = _is_host(a, b)
        ctx = _ctx_of(a, b)
        da, db = upload(a, ctx), upload(b, ctx)
        o = _new()
        check(_L.rq_mask_or(ctx.handle, da.handle, db.handle, C.byref(o)))
        return _out(DeviceMask(o, ctx), host)

    @staticmethod
    def not_mask(a):
        """masks::not_mask (mask_ops.cpp:239-265)."""
        host = _is_host(a)
        ctx = _ctx_of(a)
        da = upload(a, ctx)
        o = _new()
        check(_L.rq_mask_not(ctx.handle, da.handle, C.byref(o)))
        return _out(DeviceMask(o, ctx), host)


class X:
    """Aggregate expressions for agg.group_aggregate_exprs — the runner's
    arith / arith_scalar plan nodes (align.cpp:495-508, :571-596) as a
    left-deep chain of at most 3 terms:
        X.col(c)                    a column
        X.col(c).scalar(k, op)      c op k   (reversed=True: k op c)
        x.arith(y, op)              x op y   (y a single term)
        X.count()                   COUNT(*)
    """

    def __init__(self, terms, ops):
        self.terms, self.ops = terms, ops

    @staticmethod
    def col(c):
        return X([[c, -1, False, 0]], [])

    @staticmethod
    def count():
        return X([], [])

    def scalar(self, k, op, reversed=False):
        assert len(self.terms) == 1 and self.terms[0][1] == -1, "scalar op applies to a bare column term"
        c = self.terms[0][0]
        return X([[c, H.BINOP_NAMES.get(op, op), bool(reversed), k]], [])

    def arith(self, other, op):
        assert len(other.terms) == 1, "right operand must be a single term (left-deep chains)"
        return X(self.terms + other.terms, self.ops + [H.BINOP_NAMES.get(op, op)])


class Catalog:
    """runq::query::Catalog (runner.hpp:14-28) of device-resident columns;
    run_plan executes a reference JSON plan on the device (runner.cpp:86-373)."""

    def __init__(self, ctx: Context = None):
        self.ctx = _ctx(ctx)
        self.h = C.c_void_p()
        check(_L.rq_catalog_create(C.byref(self.h)))
        self._cols = []

    def add_column(self, table, name, col, dict=None, dict_name=None, is_date=False):
        dc = upload(col, self.ctx)
        self._cols.append(dc)
        strs = [s.encode() for s in (dict or [])]
        arr = (C.c_char_p * max(1, len(strs)))(*strs)
        check(_L.rq_catalog_add_column(self.h, table.encode(), name.encode(), dc.handle, arr, len(strs),
                                       dict_name.encode() if dict_name else None, int(is_date)))

    def run_plan(self, plan_json: str):
        """-> (dict column name -> numpy values, rows, fused GroupAgg nodes)."""
        r = C.c_void_p()
        check(_L.rq_run_plan(self.ctx.handle, self.h, plan_json.encode(), C.byref(r)))
        try:
            nc, rows, fused = C.c_int32(), C.c_int64(), C.c_int32()
            check(_L.rq_result_info(r, C.byref(nc), C.byref(rows), C.byref(fused)))
            out = {}
            for i in range(nc.value):
                name, arr = C.c_char_p(), C.c_void_p()
                check(_L.rq_result_column(r, i, C.byref(name), C.byref(arr)))
                out[name.value.decode()] = DeviceArray(arr, self.ctx).download()
            return out, int(rows.value), int(fused.value)
        finally:
            _L.rq_result_free(r)

    def __del__(self):
        if getattr(self, "h", None):
            _L.rq_catalog_destroy(self.h)
            self.h = None


class joins:
    @staticmethod
    def hash_build_probe(build_values, probe_values):
        """joins::hash_build_probe (join.cpp:167-181) -> (build_pos, probe_pos) numpy arrays."""
        ctx = _ctx_of(build_values, probe_values)
        db, dp = upload(np.asarray(build_values), ctx), upload(np.asarray(probe_values), ctx)
        ob, op = C.c_void_p(), C.c_void_p()
        check(_L.rq_hash_build_probe(ctx.handle, db.handle, dp.handle, C.byref(ob), C.byref(op)))
        return DeviceArray(ob, ctx).download(), DeviceArray(op, ctx).download()

    @staticmethod
    def get_join_index(left, right):
        """joins::get_join_index (join.cpp:183-238) -> (left side, right side,
        cardinality); a side is ("rows", rows) or ("rle", v, s, e) (numpy)."""
        ctx = _ctx_of(left, right)
        dl, dr = upload(left, ctx), upload(right, ctx)
        lo, ro, card = H.JoinSide(), H.JoinSide(), C.c_int64()
        check(_L.rq_get_join_index(ctx.handle, dl.handle, dr.handle, C.byref(lo), C.byref(ro), C.byref(card)))

        def side(j):
            if j.is_rle:
                return ("rle",) + tuple(DeviceArray(C.c_void_p(p), ctx).download() for p in (j.v, j.s, j.e))
            return ("rows", DeviceArray(C.c_void_p(j.rows), ctx).download())
        return side(lo), side(ro), int(card.value)

    @staticmethod
    def apply_join_index(col, side):
        """joins::apply_join_index (join.cpp:363-366) of a side ("rows", rows) / ("rle", v, s, e)."""
        host = _is_host(col)
        ctx = _ctx_of(col)
        dc = upload(col, ctx)
        arrs = [upload(np.ascontiguousarray(a, dtype=np.int64), ctx) for a in side[1:]]
        j = H.JoinSide()
        j.is_rle = 1 if side[0] == "rle" else 0
        if j.is_rle:
            j.v, j.s, j.e = (a.handle.value for a in arrs)
        else:
            j.rows = arrs[0].handle.value
        o = _new()
        check(_L.rq_apply_join_index(ctx.handle, dc.handle, C.byref(j), C.byref(o)))
        return _out(DeviceColumn(o, ctx), host)

    @staticmethod
    def semi_join_mask(probe, build):
        """joins::semi_join_mask (join.cpp:368-406): probe rows whose key occurs in build."""
        host = _is_host(probe, build)
        ctx = _ctx_of(probe, build)
        dp, db = upload(probe, ctx), upload(build, ctx)
        o = _new()
        check(_L.rq_semi_join_mask(ctx.handle, dp.handle, db.handle, C.byref(o)))
        return _out(DeviceMask(o, ctx), host)


class Comm:
    """rq_comm_t: the ranks of a row-range sharded table.

    ``Comm.nccl(ctx, uid, nranks, rank)`` — one rank per GPU over NCCL (rank 0
    makes ``uid = Comm.unique_id()`` and the launcher broadcasts it);
    ``Comm.host(ctx, nranks, rank, allgather)`` — the host transport, where
    ``allgather(bytes) -> list[bytes]`` (one entry per rank) moves the
    packets, e.g. over torch.distributed gloo with several ranks on one GPU."""

    def __init__(self, handle, ctx, keep=None):
        self.handle, self.ctx, self._keep = handle, ctx, keep

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(_L.rq_comm_unique_id(buf, 128))
        return buf.raw

    @classmethod
    def nccl(cls, ctx: Context, uid: bytes, nranks: int, rank: int) -> "Comm":
        h = C.c_void_p()
        buf = C.create_string_buffer(bytes(uid), 128)
        check(_L.rq_comm_init_nccl(ctx.handle, buf, nranks, rank, C.byref(h)))
        return cls(h, ctx)

    @classmethod
    def host(cls, ctx: Context, nranks: int, rank: int, allgather) -> "Comm":
        from ._lib import HOST_ALLGATHER_FN

        def cb(send, nbytes, recv, user):
            try:
                parts = allgather(C.string_at(send, nbytes) if nbytes else b"")
                blob = b"".join(parts)
                assert len(blob) == nbytes * nranks
                if blob:
                    C.memmove(recv, blob, len(blob))
                return 0
            except Exception:  # noqa: BLE001 — reported as RQ_NCCL by the library
                return 1
        fn = HOST_ALLGATHER_FN(cb)
        h = C.c_void_p()
        check(_L.rq_comm_init_host(ctx.handle, nranks, rank, fn, None, C.byref(h)))
        return cls(h, ctx, keep=fn)

    def info(self):
        n, r, t = C.c_int32(), C.c_int32(), C.c_int32()
        check(_L.rq_comm_info(self.handle, C.byref(n), C.byref(r), C.byref(t)))
        return int(n.value), int(r.value), ("nccl", "host")[t.value]

    def __del__(self):
        if getattr(self, "handle", None):
            _L.rq_comm_destroy(self.handle)
            self.handle = None


def _agg_result(dt, i, f):
    return float(f.value) if dt.value == H.F64 else int(i.value)


class agg:
    SUM, COUNT, MIN, MAX, AVG, STD, VAR = range(7)

    class GroupingResult:
        """agg::GroupingResult (groupby.hpp:12-18)."""

        def __init__(self, inverse, n_groups, keys, shape, total_size):
            self.inverse, self.n_groups, self.keys, self.shape, self.total_size = \
                inverse, n_groups, keys, shape, total_size

    @staticmethod
    def group(keys: Sequence) -> "agg.GroupingResult":
        """agg::group (groupby.cpp:46-50): align_many + unique_with_inverse."""
        host = _is_host(*keys)
        ctx = _ctx_of(*keys)
        dk = [upload(k, ctx) for k in keys]
        arr = (C.c_void_p * len(dk))(*[d.handle.value for d in dk])
        ko = (C.c_void_p * len(dk))()
        k, n, ps, pe, pp = _shape_outs()
        inv, ng = _new(), C.c_int64()
        check(_L.rq_group(ctx.handle, arr, len(dk), C.byref(k), C.byref(n), C.byref(ps), C.byref(pe), C.byref(pp),
                          C.byref(inv), ko, C.byref(ng)))
        return agg.GroupingResult(_out(DeviceArray(inv, ctx), host), int(ng.value),
                                  [_out(DeviceArray(C.c_void_p(ko[i]), ctx), host) for i in range(len(dk))],
                                  Shape._from(k, n, ps, pe, pp, ctx, host), dk[0].total_size)

    @staticmethod
    def group_on_arrays(shape: Shape, key_values: Sequence, total_size: int) -> "agg.GroupingResult":
        """agg::group_on_arrays (groupby.cpp:33-44)."""
        host = _is_host(*key_values)
        ctx = _ctx_of(*key_values)
        dk = [_arr_in(k, ctx) for k in key_values]
        arr = (C.c_void_p * max(1, len(dk)))(*[d.handle.value for d in dk])
        ko = (C.c_void_p * max(1, len(dk)))()
        inv, ng = _new(), C.c_int64()
        check(_L.rq_group_on_arrays(ctx.handle, arr, len(dk), C.byref(inv), ko, C.byref(ng)))
        return agg.GroupingResult(_out(DeviceArray(inv, ctx), host), int(ng.value),
                                  [_out(DeviceArray(C.c_void_p(ko[i]), ctx), host) for i in range(len(dk))],
                                  shape, total_size)

    @staticmethod
    def aggregate_array(shape: Shape, values, g: "agg.GroupingResult", fn):
        """agg::aggregate_array (groupby.cpp:67-135)."""
        fn = H.AGG_NAMES.get(fn, fn)
        host = _is_host(values, g.inverse)
        ctx = _ctx_of(values, g.inverse)
        v, inv = _arr_in(values, ctx), _arr_in(g.inverse, ctx, np.int64)
        o = _new()
        check(_L.rq_aggregate_array(ctx.handle, *shape._args(ctx), v.handle, inv.handle, C.c_int64(g.n_groups),
                                    C.c_int32(fn), C.byref(o)))
        return _out(DeviceArray(o, ctx), host)

    @staticmethod
    def aggregate(data, g: "agg.GroupingResult", fn):
        """agg::aggregate (groupby.cpp:137-142): data must decompose onto g's shape."""
        sh, vals = compute.decompose(data)
        a, b = g.shape, sh
        same = a.kind == b.kind and (
            (a.kind == "dense" and a.n == b.n) or
            (a.kind == "run" and np.array_equal(_host_arr(a.s), _host_arr(b.s)) and
             np.array_equal(_host_arr(a.e), _host_arr(b.e))) or
            (a.kind == "point" and np.array_equal(_host_arr(a.p), _host_arr(b.p))))
        if not same:
            raise RqError(1, "aggregate: data shape differs from grouping shape")
        return agg.aggregate_array(sh, vals, g, fn)

    @staticmethod
    def aggregate_all(data, fn, comm: Comm = None):
        """agg::aggregate_all (groupby.cpp:164-172) -> python int (i64) or float (f64).
        With `comm`: this rank's shard, merged over the communicator."""
        fn = H.AGG_NAMES.get(fn, fn)
        ctx = _ctx_of(data)
        dd = upload(data, ctx)
        dt, i, f = C.c_int32(), C.c_int64(), C.c_double()
        if comm is not None:
            check(_L.rq_aggregate_all_sharded(ctx.handle, comm.handle, dd.handle, fn, C.byref(dt), C.byref(i),
                                              C.byref(f)))
            return _agg_result(dt, i, f)
        check(_L.rq_aggregate_all(ctx.handle, dd.handle, fn, C.byref(dt), C.byref(i), C.byref(f)))
        return _agg_result(dt, i, f)

    @staticmethod
    def group_aggregate(keys: Sequence, data: Sequence, fns: Sequence, normalize: bool = False, comm: Comm = None):
        """agg::group_aggregate (groupby.cpp:144-162) -> (keys list, values list, n_groups).
        normalize=True: the query runner's GroupAgg (normalize_basic on every
        input first, runner.cpp:306-336), composites folded without expansion."""
        fns = [H.AGG_NAMES.get(f, f) for f in fns]
        fn_c = _L.rq_group_aggregate_normalized if normalize else _L.rq_group_aggregate
        host = _is_host(*keys, *data)
        ctx = _ctx_of(*keys, *data)
        dk = [upload(k, ctx) for k in keys]
        dd = [upload(d, ctx) for d in data]
        karr = (C.c_void_p * max(1, len(dk)))(*[k.handle.value for k in dk])
        darr = (C.c_void_p * max(1, len(dd)))(*[d.handle.value for d in dd])
        farr = (C.c_int32 * max(1, len(fns)))(*fns)
        ok = (C.c_void_p * max(1, len(dk)))()
        ov = (C.c_void_p * max(1, len(dd)))()
        ng = C.c_int64()
        if comm is not None:
            check(_L.rq_group_aggregate_sharded(ctx.handle, comm.handle, karr, len(dk), darr, farr, len(dd),
                                                int(normalize), C.byref(ng), ok, ov))
        else:
            check(fn_c(ctx.handle, karr, len(dk), darr, farr, len(dd), C.byref(ng), ok, ov))
        ks = [_out(DeviceArray(C.c_void_p(ok[i]), ctx), host) for i in range(len(dk))]
        vs = [_out(DeviceArray(C.c_void_p(ov[i]), ctx), host) for i in range(len(dd))]
        return ks, vs, int(ng.value)

    @staticmethod
    def group_aggregate_exprs(mask, keys: Sequence, exprs: Sequence, fns: Sequence, where: Sequence = (),
                              comm: Comm = None):
        """The runner's Filter → expressions → GroupAgg (runner.cpp:243-336)
        in one call: operands filtered by `mask` (None: no WHERE) and by the
        conjuncts `where` — (col, op, k) or (col, "in", [k...]) — each X
        expression evaluated, group_aggregate(normalize) over `keys` (empty:
        one global group). Returns (keys list, values list, n_groups, fused)."""
        return PreparedExprs(mask, keys, exprs, fns, where, comm)()

    @staticmethod
    def prepare_exprs(mask, keys: Sequence, exprs: Sequence, fns: Sequence, where: Sequence = (),
                      comm: Comm = None) -> "PreparedExprs":
        """group_aggregate_exprs with its arguments marshalled once: calling
        the result runs the query again (a repeated plan on the same device
        handles is replayed by the library as one CUDA graph)."""
        return PreparedExprs(mask, keys, exprs, fns, where, comm)

    @staticmethod
    def aggregate_binop(a, b, op, fn, comm: Comm = None):
        """Fused aggregate_all(arith(a, b, op), fn) — one pass, no materialised fragments."""
        op = H.BINOP_NAMES.get(op, op)
        fn = H.AGG_NAMES.get(fn, fn)
        ctx = _ctx_of(a, b)
        da, db = upload(a, ctx), upload(b, ctx)
        dt, i, f = C.c_int32(), C.c_int64(), C.c_double()
        if comm is not None:
            check(_L.rq_aggregate_binop_sharded(ctx.handle, comm.handle, da.handle, db.handle, op, fn, C.byref(dt),
                                                C.byref(i), C.byref(f)))
            return _agg_result(dt, i, f)
        check(_L.rq_aggregate_binop(ctx.handle, da.handle, db.handle, op, fn, C.byref(dt), C.byref(i), C.byref(f)))
        return _agg_result(dt, i, f)

    @staticmethod
    def filtered_aggregate_binop(c, k, cmp, a, b, op, fn, comm: Comm = None):
        """aggregate_all(arith(filter(a,m), filter(b,m), op), fn), m = compare_scalar(c, k, cmp)."""
        op = H.BINOP_NAMES.get(op, op)
        cmp = H.BINOP_NAMES.get(cmp, cmp)
        fn = H.AGG_NAMES.get(fn, fn)
        ctx = _ctx_of(c, a, b)
        dc, da, db = upload(c, ctx), upload(a, ctx), upload(b, ctx)
        dt, i, f = C.c_int32(), C.c_int64(), C.c_double()
        if comm is not None:
            check(_L.rq_filtered_aggregate_binop_sharded(ctx.handle, comm.handle, dc.handle, H.make_scalar(k), cmp,
                                                         da.handle, db.handle, op, fn, C.byref(dt), C.byref(i),
                                                         C.byref(f)))
            return _agg_result(dt, i, f)
        check(_L.rq_filtered_aggregate_binop(ctx.handle, dc.handle, H.make_scalar(k), cmp, da.handle, db.handle,
                                             op, fn, C.byref(dt), C.byref(i), C.byref(f)))
        return _agg_result(dt, i, f)


def _prepared_call(fnc, args, keep, dt, i, f):
    """A fused scalar call with its ctypes arguments built once: calling it
    runs the query again on the same device handles (`keep` holds them)."""
    def run():
        check(fnc(*args))
        return _agg_result(dt, i, f)
    run.handles = keep
    return run


def prepare_binop(a, b, op, fn, comm: Comm = None):
    """agg.aggregate_binop with its arguments marshalled once (the call a
    repeated query makes): returns a callable running rq_aggregate_binop(_sharded)."""
    op = H.BINOP_NAMES.get(op, op)
    fn = H.AGG_NAMES.get(fn, fn)
    ctx = _ctx_of(a, b)
    da, db = upload(a, ctx), upload(b, ctx)
    dt, i, f = C.c_int32(), C.c_int64(), C.c_double()
    out = (C.byref(dt), C.byref(i), C.byref(f))
    if comm is not None:
        return _prepared_call(_L.rq_aggregate_binop_sharded,
                              (ctx.handle, comm.handle, da.handle, db.handle, op, fn) + out, (da, db, comm), dt, i, f)
    return _prepared_call(_L.rq_aggregate_binop, (ctx.handle, da.handle, db.handle, op, fn) + out, (da, db), dt, i, f)


def prepare_filtered_binop(c, k, cmp, a, b, op, fn, comm: Comm = None):
    """agg.filtered_aggregate_binop with its arguments marshalled once:
    returns a callable running rq_filtered_aggregate_binop(_sharded)."""
    op = H.BINOP_NAMES.get(op, op)
    cmp = H.BINOP_NAMES.get(cmp, cmp)
    fn = H.AGG_NAMES.get(fn, fn)
    ctx = _ctx_of(c, a, b)
    dc, da, db = upload(c, ctx), upload(a, ctx), upload(b, ctx)
    ks = H.make_scalar(k)
    dt, i, f = C.c_int32(), C.c_int64(), C.c_double()
    out = (C.byref(dt), C.byref(i), C.byref(f))
    if comm is not None:
        return _prepared_call(_L.rq_filtered_aggregate_binop_sharded,
                              (ctx.handle, comm.handle, dc.handle, ks, cmp, da.handle, db.handle, op, fn) + out,
                              (dc, da, db, ks, comm), dt, i, f)
    return _prepared_call(_L.rq_filtered_aggregate_binop,
                          (ctx.handle, dc.handle, ks, cmp, da.handle, db.handle, op, fn) + out, (dc, da, db, ks),
                          dt, i, f)


agg.prepare_binop = staticmethod(prepare_binop)
agg.prepare_filtered_binop = staticmethod(prepare_filtered_binop)


def shard_host_column(col: H.Column, lo: int, hi: int) -> H.Column:
    """rq_shard_host_column: rows [lo, hi) as a standalone shard (host only)."""
    img, keep = H.column_image(col)
    out = H.HostColumn()
    check(_L.rq_shard_host_column(C.byref(img), lo, hi, C.byref(out)))
    try:
        return H.column_from_malloc_image(out)
    finally:
        _L.rq_host_column_free(C.byref(out))


class PreparedExprs:
    """rq_group_aggregate_where(_sharded) with its C arguments built once (the
    device columns the plan names are uploaded once and kept alive)."""

    def __init__(self, mask, keys: Sequence, exprs: Sequence, fns: Sequence, where: Sequence = (),
                 comm: Comm = None):
        fns = [H.AGG_NAMES.get(f, f) for f in fns]
        cols = [t[0] for x in exprs for t in x.terms] + [w[0] for w in where]
        self.host = _is_host(*keys, *cols, *([mask] if mask is not None else []))
        ctx = self.ctx = _ctx_of(*keys, *cols, *([mask] if mask is not None else []))
        dm = upload(mask, ctx) if mask is not None else None
        dk = [upload(k, ctx) for k in keys]
        arr = (H.Expr * len(exprs))()
        keep = [dm, dk]
        uploaded = {}  # one device column per distinct operand object

        def up(c):
            if id(c) not in uploaded:
                uploaded[id(c)] = (c, upload(c, ctx))
            return uploaded[id(c)][1]
        for i, x in enumerate(exprs):
            arr[i].n_terms = len(x.terms)
            for j, op in enumerate(x.ops):
                arr[i].ops[j] = op
            for j, (c, op, rev, k) in enumerate(x.terms):
                dc = up(c)
                keep.append(dc)
                arr[i].terms[j].col = dc.handle.value
                arr[i].terms[j].op = op
                arr[i].terms[j].reversed = int(rev)
                arr[i].terms[j].k = H.make_scalar(k)
        warr = (H.Pred * max(1, len(where)))()
        for i, w in enumerate(where):
            col, op, k = w
            warr[i].col = up(col).handle.value
            if isinstance(op, str) and op.lower() == "in":
                lst = (H.Scalar * len(k))(*[H.make_scalar(x) for x in k])
                keep.append(lst)
                warr[i].op, warr[i].n_in, warr[i].in_list = 0, len(k), lst
                warr[i].k = H.make_scalar(0)
            else:
                warr[i].op, warr[i].n_in = H.BINOP_NAMES.get(op, op), 0
                warr[i].k = H.make_scalar(k)
        keep.extend(uploaded.values())
        self._keep = keep
        self.nk, self.ne, self.nw = len(dk), len(exprs), len(where)
        self._args = (warr, len(where), dm.handle if dm is not None else None,
                      (C.c_void_p * max(1, len(dk)))(*[k.handle.value for k in dk]), len(dk), arr,
                      (C.c_int32 * len(fns))(*fns), len(exprs))
        self.comm = comm

    def __call__(self):
        ok = (C.c_void_p * max(1, self.nk))()
        ov = (C.c_void_p * self.ne)()
        ng, fused = C.c_int64(), C.c_int32()
        warr, nw, dm, karr, nk, arr, farr, ne = self._args
        if self.comm is not None:
            check(_L.rq_group_aggregate_where_sharded(self.ctx.handle, self.comm.handle, warr, nw, dm, karr, nk, arr,
                                                      farr, ne, C.byref(ng), ok, ov, C.byref(fused)))
        else:
            check(_L.rq_group_aggregate_where(self.ctx.handle, warr, nw, dm, karr, nk, arr, farr, ne, C.byref(ng), ok,
                                              ov, C.byref(fused)))
        ks = [_out(DeviceArray(C.c_void_p(ok[i]), self.ctx), self.host) for i in range(self.nk)]
        vs = [_out(DeviceArray(C.c_void_p(ov[i]), self.ctx), self.host) for i in range(self.ne)]
        return ks, vs, int(ng.value), bool(fused.value)
