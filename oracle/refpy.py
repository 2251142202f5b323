"""TEST INFRASTRUCTURE ONLY — Python access to the two checkers:

* ``Ref``: the UNMODIFIED reference library (oracle/_ref/librunq_ref.so, built
  from /root/reference/proj/core/src by oracle/Makefile) through the extern "C"
  shim ``oracle/ref_shim.cpp``. Same operator names and argument meaning as
  the product's ``paper_2506_10092_b200.runq`` so parity tests read alike.
* ``Orq``: the plain-C restatement (oracle/liboracle.so, runq_oracle.c).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2506_10092_b200 import host as H

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "librunq_ref.so")
ORQ_SO = os.path.join(HERE, "liboracle.so")
REFERENCE_SRC = "/root/reference/proj/core/src"


def build(quiet: bool = True) -> None:
    """Builds liboracle.so always and _ref/librunq_ref.so when the reference
    sources are present (this container); the GPU box uses prebuilt files."""
    targets = ["liboracle.so"]
    if os.path.isdir(REFERENCE_SRC):
        targets.append("ref")
    subprocess.run(["make", "-C", HERE, "-j8", *targets], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


class RefHostArray(C.Structure):
    _fields_ = [("dtype", C.c_int32), ("_pad", C.c_int32), ("n", C.c_int64), ("data", C.c_void_p)]


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def _take(ptr, n, dt):
    if n == 0 or not ptr:
        return np.empty(0, dtype=dt)
    buf = (C.c_char * (n * np.dtype(dt).itemsize)).from_address(ptr)
    return np.frombuffer(bytes(buf), dtype=dt).copy()


class RefJoinSide(C.Structure):
    _fields_ = [("is_rle", C.c_int32), ("n", C.c_int64), ("rows", C.POINTER(C.c_int64)), ("v", C.POINTER(C.c_int64)),
                ("s", C.POINTER(C.c_int64)), ("e", C.POINTER(C.c_int64))]


class RefCatalog:
    """runq::query::Catalog of the reference built from column images, and
    runq::query::run in Compressed mode over it (runner.cpp:457-520)."""

    def __init__(self, ref):
        self.ref = ref
        self.h = C.c_void_p()
        ref._check(ref.lib.ref_catalog_create(C.byref(self.h)))
        self._keep = []

    def add_column(self, table, name, col, dict=None, dict_name=None, is_date=False):
        img, keep = H.column_image(col)
        self._keep.append((img, keep))
        strs = [s.encode() for s in (dict or [])]
        arr = (C.c_char_p * max(1, len(strs)))(*strs)
        self.ref._check(self.ref.lib.ref_catalog_add_column(
            self.h, table.encode(), name.encode(), C.byref(img), arr, len(strs),
            dict_name.encode() if dict_name else None, int(is_date)))

    def run_plan(self, plan_json: str):
        lib = self.ref.lib
        r = C.c_void_p()
        self.ref._check(lib.ref_run_plan(self.h, plan_json.encode(), C.byref(r)))
        try:
            nc, rows = C.c_int32(), C.c_int64()
            self.ref._check(lib.ref_result_info(r, C.byref(nc), C.byref(rows)))
            out = {}
            for i in range(nc.value):
                name, dt, data, n = C.c_char_p(), C.c_int32(), C.c_void_p(), C.c_int64()
                self.ref._check(lib.ref_result_column(r, i, C.byref(name), C.byref(dt), C.byref(data), C.byref(n)))
                npdt = H.DTYPES[dt.value]
                buf = (C.c_char * (n.value * np.dtype(npdt).itemsize)).from_address(data.value) if n.value else b""
                out[name.value.decode()] = np.frombuffer(bytes(buf), dtype=npdt).copy()
            return out
        finally:
            lib.ref_result_free(r)

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.ref_catalog_free(self.h)
            self.h = None


class Ref:
    """The reference operator API (runq::compute / enc / masks / agg)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: build with `make -C oracle ref`")
        self.lib = C.CDLL(path)
        self.lib.ref_last_error.restype = C.c_char_p

    def _check(self, st):
        if st != 0:
            raise RefError(st, self.lib.ref_last_error().decode(errors="replace"))

    def _arr(self, a: RefHostArray) -> np.ndarray:
        out = _take(a.data, a.n, H.DTYPES[a.dtype])
        self.lib.ref_free_array(C.byref(a))
        return out

    def _col(self, h: H.HostColumn) -> H.Column:
        c = H.column_from_malloc_image(h)
        self.lib.ref_free_column(C.byref(h))
        return c

    def _mask(self, h: H.HostMask) -> H.Mask:
        m = H.mask_from_malloc_image(h)
        self.lib.ref_free_mask(C.byref(h))
        return m

    @staticmethod
    def _p(a):
        a = np.ascontiguousarray(np.asarray(a, dtype=np.int64))
        return a, (a.ctypes.data if a.size else None), a.shape[0]

    # --- enc ---
    def range_intersect(self, s1, e1, s2, e2):
        (a1, p1, n1), (b1, q1, _), (a2, p2, n2), (b2, q2, _) = map(self._p, (s1, e1, s2, e2))
        outs = [RefHostArray() for _ in range(4)]
        self._check(self.lib.ref_range_intersect(C.c_void_p(p1), C.c_void_p(q1), C.c_int64(n1),
                                                 C.c_void_p(p2), C.c_void_p(q2), C.c_int64(n2),
                                                 *[C.byref(o) for o in outs]))
        return tuple(self._arr(o) for o in outs)

    def _pts(self, fn, p, s, e):
        (a, pp, np_), (b, sp, nr), (c, ep, _) = map(self._p, (p, s, e))
        outs = [RefHostArray() for _ in range(3)]
        self._check(fn(C.c_void_p(pp), C.c_int64(np_), C.c_void_p(sp), C.c_void_p(ep), C.c_int64(nr),
                       *[C.byref(o) for o in outs]))
        return tuple(self._arr(o) for o in outs)

    def idx_in_rle(self, p, s, e):
        return self._pts(self.lib.ref_idx_in_rle, p, s, e)

    def rle_contain_idx(self, p, s, e):
        return self._pts(self.lib.ref_rle_contain_idx, p, s, e)

    def idx_in_idx(self, p1, p2):
        (a, pa, na), (b, pb, nb) = map(self._p, (p1, p2))
        outs = [RefHostArray() for _ in range(3)]
        self._check(self.lib.ref_idx_in_idx(C.c_void_p(pa), C.c_int64(na), C.c_void_p(pb), C.c_int64(nb),
                                            *[C.byref(o) for o in outs]))
        return tuple(self._arr(o) for o in outs)

    def bucketize(self, x, b, right):
        (a, pa, na), (bb, pb, nb) = map(self._p, (x, b))
        o = RefHostArray()
        self._check(self.lib.ref_bucketize(C.c_void_p(pa), C.c_int64(na), C.c_void_p(pb), C.c_int64(nb),
                                           C.c_int32(1 if right else 0), C.byref(o)))
        return self._arr(o)

    def plain_mask_to_rle(self, m):
        img, keep = H.mask_image(m)
        out = H.HostMask()
        self._check(self.lib.ref_plain_mask_to_rle(C.byref(img), C.byref(out)))
        return self._mask(out)

    def plain_mask_to_index(self, m):
        img, keep = H.mask_image(m)
        out = H.HostMask()
        self._check(self.lib.ref_plain_mask_to_index(C.byref(img), C.byref(out)))
        return self._mask(out)

    def compact_rle(self, c):
        img, keep = H.column_image(c)
        out = H.HostColumn()
        self._check(self.lib.ref_compact_rle(C.byref(img), C.byref(out)))
        return self._col(out)

    def plain_to_rle(self, c):
        img, keep = H.column_image(c)
        out = H.HostColumn()
        self._check(self.lib.ref_plain_to_rle(C.byref(img), C.byref(out)))
        return self._col(out)

    def plain_to_rle_index(self, c, min_run):
        img, keep = H.column_image(c)
        out = H.HostColumn()
        self._check(self.lib.ref_plain_to_rle_index(C.byref(img), C.c_int64(min_run), C.byref(out)))
        return self._col(out)

    def plain_to_plain_index(self, c, trim):
        img, keep = H.column_image(c)
        out = H.HostColumn()
        self._check(self.lib.ref_plain_to_plain_index(C.byref(img), C.c_double(trim), C.byref(out)))
        return self._col(out)

    # --- io (ingest.hpp:56-62) ---
    def choose_encoding(self, c, cfg=None):
        img, keep = H.column_image(c)
        out = H.EncodingChoice()
        self._check(self.lib.ref_choose_encoding(C.byref(img), C.byref(cfg) if cfg is not None else None,
                                                 C.byref(out)))
        return out

    def encode(self, c, choice):
        img, keep = H.column_image(c)
        out = H.HostColumn()
        self._check(self.lib.ref_encode(C.byref(img), C.byref(choice), C.byref(out)))
        return self._col(out)

    def sort_table(self, cols, by):
        imgs = [H.column_image(c) for c in cols]
        arr = (H.HostColumn * len(cols))(*[i for i, _ in imgs])
        outs = (H.HostColumn * len(cols))()
        bys = (C.c_int32 * len(by))(*by)
        self._check(self.lib.ref_sort_table(arr, C.c_int32(len(cols)), bys, C.c_int32(len(by)), outs))
        return [self._col(o) for o in outs]

    # --- column model ---
    def roundtrip(self, c):
        img, keep = H.column_image(c)
        out = H.HostColumn()
        self._check(self.lib.ref_roundtrip(C.byref(img), C.byref(out)))
        return self._col(out)

    def validate(self, c) -> int:
        img, keep = H.column_image(c)
        return int(self.lib.ref_validate(C.byref(img)))

    def decode_values(self, c):
        img, keep = H.column_image(c)
        o = RefHostArray()
        self._check(self.lib.ref_decode_values(C.byref(img), C.byref(o)))
        return self._arr(o)

    def dump_column(self, c) -> bytes:
        """runq::dump_column (column.cpp:513-563): JSON header line + raw arrays."""
        img, keep = H.column_image(c)
        o = RefHostArray()
        self._check(self.lib.ref_dump_column(C.byref(img), C.byref(o)))
        try:
            return C.string_at(o.data, o.n) if o.n else b""
        finally:
            self.lib.ref_free_array(C.byref(o))

    def normalize_basic(self, c):
        img, keep = H.column_image(c)
        out = H.HostColumn()
        self._check(self.lib.ref_normalize_basic(C.byref(img), C.byref(out)))
        return self._col(out)

    # --- compute ---
    def align(self, a, b):
        ia, ka = H.column_image(a)
        ib, kb = H.column_image(b)
        kind = C.c_int32()
        outs = [RefHostArray() for _ in range(5)]
        self._check(self.lib.ref_align(C.byref(ia), C.byref(ib), C.byref(kind), *[C.byref(o) for o in outs]))
        res = {"kind": int(kind.value)}
        for name, o in zip(("s", "e", "p", "v1", "v2"), outs):
            present = bool(o.data)
            arr = self._arr(o)
            res[name] = arr if present else None
        return res

    def arith(self, a, b, op):
        op = H.BINOP_NAMES.get(op, op)
        ia, ka = H.column_image(a)
        ib, kb = H.column_image(b)
        out = H.HostColumn()
        self._check(self.lib.ref_arith(C.byref(ia), C.byref(ib), C.c_int32(op), C.byref(out)))
        return self._col(out)

    def compare(self, a, b, op):
        op = H.BINOP_NAMES.get(op, op)
        ia, ka = H.column_image(a)
        ib, kb = H.column_image(b)
        out = H.HostMask()
        self._check(self.lib.ref_compare(C.byref(ia), C.byref(ib), C.c_int32(op), C.byref(out)))
        return self._mask(out)

    def arith_scalar(self, a, k, op, reversed=False):
        op = H.BINOP_NAMES.get(op, op)
        ia, ka = H.column_image(a)
        out = H.HostColumn()
        self.lib.ref_arith_scalar.argtypes = [C.c_void_p, H.Scalar, C.c_int32, C.c_int32, C.c_void_p]
        self._check(self.lib.ref_arith_scalar(C.byref(ia), H.make_scalar(k), op, 1 if reversed else 0,
                                               C.byref(out)))
        return self._col(out)

    def compare_scalar(self, a, k, op, reversed=False):
        op = H.BINOP_NAMES.get(op, op)
        ia, ka = H.column_image(a)
        out = H.HostMask()
        self.lib.ref_compare_scalar.argtypes = [C.c_void_p, H.Scalar, C.c_int32, C.c_int32, C.c_void_p]
        self._check(self.lib.ref_compare_scalar(C.byref(ia), H.make_scalar(k), op, 1 if reversed else 0,
                                                 C.byref(out)))
        return self._mask(out)

    def filter(self, a, m):
        ia, ka = H.column_image(a)
        im, km = H.mask_image(m)
        out = H.HostColumn()
        self._check(self.lib.ref_filter(C.byref(ia), C.byref(im), C.byref(out)))
        return self._col(out)

    def hash_build_probe(self, build_values, probe_values):
        """joins::hash_build_probe (join.cpp:167-181) -> (build_pos, probe_pos)."""
        b = np.ascontiguousarray(build_values)
        p = np.ascontiguousarray(probe_values)
        bp, pp, n = C.POINTER(C.c_int64)(), C.POINTER(C.c_int64)(), C.c_int64()
        self._check(self.lib.ref_hash_build_probe(
            b.ctypes.data if b.size else None, H.dtype_code(b), b.shape[0],
            p.ctypes.data if p.size else None, H.dtype_code(p), p.shape[0], C.byref(bp), C.byref(pp), C.byref(n)))
        out = []
        for ptr in (bp, pp):
            a = np.ctypeslib.as_array(ptr, shape=(n.value,)).copy() if n.value else np.zeros(0, np.int64)
            self.lib.ref_free(C.cast(ptr, C.c_void_p))
            out.append(a)
        return out[0], out[1]

    def get_join_index(self, left, right):
        """joins::get_join_index (join.cpp:183-238) -> (left side, right side, cardinality);
        a side is ("rows", rows) or ("rle", v, s, e)."""
        il, kl = H.column_image(left)
        ir, kr = H.column_image(right)
        lo, ro, card = RefJoinSide(), RefJoinSide(), C.c_int64()
        self._check(self.lib.ref_get_join_index(C.byref(il), C.byref(ir), C.byref(lo), C.byref(ro), C.byref(card)))
        return self._side(lo), self._side(ro), int(card.value)

    def _side(self, s):
        def take(p):
            a = np.ctypeslib.as_array(p, shape=(s.n,)).copy() if s.n else np.zeros(0, np.int64)
            self.lib.ref_free(C.cast(p, C.c_void_p))
            return a
        if s.is_rle:
            return ("rle", take(s.v), take(s.s), take(s.e))
        return ("rows", take(s.rows))

    def apply_join_index(self, col, side):
        """joins::apply_join_index (join.cpp:363-366)."""
        ic, kc = H.column_image(col)
        keep = [np.ascontiguousarray(x, dtype=np.int64) for x in side[1:]]
        j = RefJoinSide()
        j.is_rle = 1 if side[0] == "rle" else 0
        j.n = len(keep[0])
        P = C.POINTER(C.c_int64)
        if j.is_rle:
            j.v, j.s, j.e = (k.ctypes.data_as(P) for k in keep)
        else:
            j.rows = keep[0].ctypes.data_as(P)
        out = H.HostColumn()
        self._check(self.lib.ref_apply_join_index(C.byref(ic), C.byref(j), C.byref(out)))
        return self._col(out)

    def semi_join_mask(self, probe, build):
        """joins::semi_join_mask (join.cpp:368-406)."""
        ip, kp = H.column_image(probe)
        ib, kb = H.column_image(build)
        out = H.HostMask()
        self._check(self.lib.ref_semi_join_mask(C.byref(ip), C.byref(ib), C.byref(out)))
        return self._mask(out)

    def and_mask(self, a, b):
        ia, ka = H.mask_image(a)
        ib, kb = H.mask_image(b)
        out = H.HostMask()
        self._check(self.lib.ref_and_mask(C.byref(ia), C.byref(ib), C.byref(out)))
        return self._mask(out)

    def or_mask(self, a, b):
        ia, ka = H.mask_image(a)
        ib, kb = H.mask_image(b)
        out = H.HostMask()
        self._check(self.lib.ref_or_mask(C.byref(ia), C.byref(ib), C.byref(out)))
        return self._mask(out)

    def not_mask(self, a):
        ia, ka = H.mask_image(a)
        out = H.HostMask()
        self._check(self.lib.ref_not_mask(C.byref(ia), C.byref(out)))
        return self._mask(out)

    def true_count(self, m) -> int:
        im, km = H.mask_image(m)
        n = C.c_int64()
        self._check(self.lib.ref_mask_true_count(C.byref(im), C.byref(n)))
        return int(n.value)

    # --- agg ---
    def aggregate_all(self, a, fn):
        fn = H.AGG_NAMES.get(fn, fn)
        ia, ka = H.column_image(a)
        dt, i, f = C.c_int32(), C.c_int64(), C.c_double()
        self._check(self.lib.ref_aggregate_all(C.byref(ia), C.c_int32(fn), C.byref(dt), C.byref(i), C.byref(f)))
        return float(f.value) if dt.value == H.F64 else int(i.value)

    def group_aggregate(self, keys, data, fns):
        fns = [H.AGG_NAMES.get(f, f) for f in fns]
        kimgs = [H.column_image(k) for k in keys]
        dimgs = [H.column_image(d) for d in data]
        karr = (H.HostColumn * max(1, len(keys)))(*[k[0] for k in kimgs])
        darr = (H.HostColumn * max(1, len(data)))(*[d[0] for d in dimgs])
        farr = (C.c_int32 * max(1, len(fns)))(*fns)
        ok = (RefHostArray * max(1, len(keys)))()
        ov = (RefHostArray * max(1, len(data)))()
        ng = C.c_int64()
        self._check(self.lib.ref_group_aggregate(karr, C.c_int32(len(keys)), darr, farr, C.c_int32(len(data)),
                                                 C.byref(ng), ok, ov))
        ks = [self._arr(ok[i]) for i in range(len(keys))]
        vs = [self._arr(ov[i]) for i in range(len(data))]
        return ks, vs, int(ng.value)

    # --- timed chains (bench cpu_baseline / --impl reference) ---
    def chain_sum_binop(self, a_shards, b_shards, nthreads, op="+"):
        op = H.BINOP_NAMES.get(op, op)
        ai = [H.column_image(c) for c in a_shards]
        bi = [H.column_image(c) for c in b_shards]
        aa = (H.HostColumn * len(ai))(*[x[0] for x in ai])
        ba = (H.HostColumn * len(bi))(*[x[0] for x in bi])
        dt, i, f, sec = C.c_int32(), C.c_int64(), C.c_double(), C.c_double()
        self._check(self.lib.ref_chain_sum_binop(aa, ba, C.c_int32(len(ai)), C.c_int32(nthreads), C.c_int32(op),
                                                 C.byref(dt), C.byref(i), C.byref(f), C.byref(sec)))
        val = float(f.value) if dt.value == H.F64 else int(i.value)
        return val, float(sec.value)

    def chain_filtered_sum(self, c_shards, a_shards, b_shards, nthreads, k, cmp="<", op="*"):
        op = H.BINOP_NAMES.get(op, op)
        cmp = H.BINOP_NAMES.get(cmp, cmp)
        ci = [H.column_image(c) for c in c_shards]
        ai = [H.column_image(c) for c in a_shards]
        bi = [H.column_image(c) for c in b_shards]
        ca = (H.HostColumn * len(ci))(*[x[0] for x in ci])
        aa = (H.HostColumn * len(ai))(*[x[0] for x in ai])
        ba = (H.HostColumn * len(bi))(*[x[0] for x in bi])
        dt, i, f, sec = C.c_int32(), C.c_int64(), C.c_double(), C.c_double()
        fn = self.lib.ref_chain_filtered_sum
        fn.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, H.Scalar, C.c_int32, C.c_int32,
                       C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        self._check(fn(ca, aa, ba, len(ci), nthreads, H.make_scalar(k), cmp, op,
                       C.byref(dt), C.byref(i), C.byref(f), C.byref(sec)))
        val = float(f.value) if dt.value == H.F64 else int(i.value)
        return val, float(sec.value)


class RefAPI:
    """The reference library behind the same namespaces as
    paper_2506_10092_b200.runq (compute / masks / agg), so one plan function
    (paper_2506_10092_b200.queries) drives both sides."""

    def __init__(self, ref: Ref = None):
        r = ref or Ref()

        class _C:
            filter = staticmethod(r.filter)
            arith = staticmethod(r.arith)
            compare = staticmethod(r.compare)
            arith_scalar = staticmethod(r.arith_scalar)
            compare_scalar = staticmethod(r.compare_scalar)
            normalize_basic = staticmethod(r.normalize_basic)

        class _M:
            and_mask = staticmethod(r.and_mask)
            or_mask = staticmethod(r.or_mask)
            not_mask = staticmethod(r.not_mask)

        class _A:
            aggregate_all = staticmethod(r.aggregate_all)

            @staticmethod
            def group_aggregate(keys, data, fns, normalize=False):
                if normalize:  # runner.cpp:306-323
                    keys = [r.normalize_basic(k) for k in keys]
                    data = [r.normalize_basic(d) for d in data]
                return r.group_aggregate(keys, data, fns)

        self.compute, self.masks, self.agg = _C, _M, _A


class Orq:
    """The plain-C restatement (runq_oracle.c)."""

    def __init__(self, path: str = ORQ_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: build with `make -C oracle liboracle.so`")
        self.lib = C.CDLL(path)
        L = self.lib
        for name in ("orq_range_intersect", "orq_idx_in_rle", "orq_rle_contain_idx", "orq_idx_in_idx",
                     "orq_plain_mask_to_rle", "orq_plain_mask_to_index", "orq_compact_rle",
                     "orq_rle_compare_scalar_i64", "orq_sum_rle_binop_i64",
                     "orq_filtered_sum_rle_idx_rle", "orq_filtered_sum_plain_idx_rle",
                     "orq_plain_to_rle_int"):
            getattr(L, name).restype = C.c_int64
        L.orq_sum_f64.restype = C.c_double

    @staticmethod
    def _p(a):
        a = np.ascontiguousarray(np.asarray(a, dtype=np.int64))
        return a

    @staticmethod
    def _ptr(a):
        return C.c_void_p(a.ctypes.data if a.size else None)

    def bucketize(self, x, b, right):
        x, b = self._p(x), self._p(b)
        out = np.empty(x.shape[0], np.int64)
        self.lib.orq_bucketize(self._ptr(x), C.c_int64(len(x)), self._ptr(b), C.c_int64(len(b)),
                               C.c_int(1 if right else 0), self._ptr(out))
        return out

    def range_intersect(self, s1, e1, s2, e2):
        s1, e1, s2, e2 = map(self._p, (s1, e1, s2, e2))
        cap = len(s1) + len(s2)
        outs = [np.empty(cap, np.int64) for _ in range(4)]
        n = self.lib.orq_range_intersect(self._ptr(s1), self._ptr(e1), C.c_int64(len(s1)), self._ptr(s2),
                                         self._ptr(e2), C.c_int64(len(s2)), *map(self._ptr, outs))
        return tuple(o[:n] for o in outs)

    def _pts(self, fn, p, s, e):
        p, s, e = map(self._p, (p, s, e))
        outs = [np.empty(len(p), np.int64) for _ in range(3)]
        n = fn(self._ptr(p), C.c_int64(len(p)), self._ptr(s), self._ptr(e), C.c_int64(len(s)),
               *map(self._ptr, outs))
        return tuple(o[:n] for o in outs)

    def idx_in_rle(self, p, s, e):
        return self._pts(self.lib.orq_idx_in_rle, p, s, e)

    def rle_contain_idx(self, p, s, e):
        return self._pts(self.lib.orq_rle_contain_idx, p, s, e)

    def idx_in_idx(self, p1, p2):
        p1, p2 = self._p(p1), self._p(p2)
        outs = [np.empty(len(p1), np.int64) for _ in range(3)]
        n = self.lib.orq_idx_in_idx(self._ptr(p1), C.c_int64(len(p1)), self._ptr(p2), C.c_int64(len(p2)),
                                    *map(self._ptr, outs))
        return tuple(o[:n] for o in outs)

    def plain_mask_to_rle(self, bits):
        bits = np.ascontiguousarray(np.asarray(bits, np.uint8))
        cap = len(bits) // 2 + 1
        s, e = np.empty(cap, np.int64), np.empty(cap, np.int64)
        n = self.lib.orq_plain_mask_to_rle(self._ptr(bits), C.c_int64(len(bits)), self._ptr(s), self._ptr(e))
        return s[:n], e[:n]

    def plain_mask_to_index(self, bits):
        bits = np.ascontiguousarray(np.asarray(bits, np.uint8))
        p = np.empty(len(bits), np.int64)
        n = self.lib.orq_plain_mask_to_index(self._ptr(bits), C.c_int64(len(bits)), self._ptr(p))
        return p[:n]

    def compact_rle(self, s, e):
        s, e = self._p(s), self._p(e)
        so, eo = np.empty(len(s), np.int64), np.empty(len(s), np.int64)
        tot = self.lib.orq_compact_rle(self._ptr(s), self._ptr(e), C.c_int64(len(s)), self._ptr(so), self._ptr(eo))
        return so, eo, int(tot)

    def plain_to_rle_int(self, values):
        """-> (s, e) of the runs of an integer storage array."""
        v = np.ascontiguousarray(values)
        s, e = np.empty(len(v), np.int64), np.empty(len(v), np.int64)
        k = self.lib.orq_plain_to_rle_int(C.c_int(H.dtype_code(v)), self._ptr(v), C.c_int64(len(v)),
                                          self._ptr(s), self._ptr(e))
        return s[:k], e[:k]

    def decode_plain_int(self, values, logical, center):
        v = np.ascontiguousarray(values)
        out = np.empty(len(v), np.int64)
        self.lib.orq_decode_plain_int(C.c_int(H.dtype_code(v)), self._ptr(v), C.c_int64(len(v)), C.c_int(logical),
                                      C.c_int(0 if center is None else 1), C.c_int64(center or 0), self._ptr(out))
        return out

    def rle_compare_scalar(self, v, s, e, op, k):
        v, s, e = self._p(v), self._p(s), self._p(e)
        so, eo = np.empty(len(s), np.int64), np.empty(len(s), np.int64)
        n = self.lib.orq_rle_compare_scalar_i64(self._ptr(v), self._ptr(s), self._ptr(e), C.c_int64(len(s)),
                                                C.c_int(H.BINOP_NAMES.get(op, op)), C.c_int64(k),
                                                self._ptr(so), self._ptr(eo))
        return so[:n], eo[:n]

    def sum_rle_binop(self, a: H.RleColumn, b: H.RleColumn, op="+") -> int:
        va, sa, ea = self._p(a.v), a.s, a.e
        vb, sb, eb = self._p(b.v), b.s, b.e
        return int(self.lib.orq_sum_rle_binop_i64(self._ptr(va), self._ptr(sa), self._ptr(ea), C.c_int64(len(sa)),
                                                  self._ptr(vb), self._ptr(sb), self._ptr(eb), C.c_int64(len(sb)),
                                                  C.c_int(H.BINOP_NAMES.get(op, op))))

    def filtered_sum(self, c, k, cmp, a: H.RleColumn, b: H.IndexColumn, op="*") -> int:
        cmp = H.BINOP_NAMES.get(cmp, cmp)
        op = H.BINOP_NAMES.get(op, op)
        av = self._p(a.v)
        bv = self._p(b.v)
        if isinstance(c, H.RleColumn):
            cv = self._p(c.v)
            return int(self.lib.orq_filtered_sum_rle_idx_rle(
                self._ptr(cv), self._ptr(c.s), self._ptr(c.e), C.c_int64(len(c.s)), C.c_int(cmp), C.c_int64(k),
                self._ptr(av), self._ptr(a.s), self._ptr(a.e), C.c_int64(len(a.s)),
                self._ptr(bv), self._ptr(b.p), C.c_int64(len(b.p)), C.c_int(op)))
        cvals = np.ascontiguousarray(c.values)
        return int(self.lib.orq_filtered_sum_plain_idx_rle(
            C.c_int(H.dtype_code(cvals)), self._ptr(cvals), C.c_int64(len(cvals)), C.c_int(c.logical),
            C.c_int(0 if c.center is None else 1), C.c_int64(c.center or 0), C.c_int(cmp), C.c_int64(k),
            self._ptr(av), self._ptr(a.s), self._ptr(a.e), C.c_int64(len(a.s)),
            self._ptr(bv), self._ptr(b.p), C.c_int64(len(b.p)), C.c_int(op)))

    def sum_f64(self, x) -> float:
        x = np.ascontiguousarray(np.asarray(x, np.float64))
        return float(self.lib.orq_sum_f64(self._ptr(x), C.c_int64(len(x))))


# ---------------------------------------------------------------------------
# row-range shard slicing for the reference arm (numpy only: the reference
# and cpu_baseline legs never load the product library)
# ---------------------------------------------------------------------------


def _slice_points(v, p, lo, hi):
    a, b = np.searchsorted(p, lo, "left"), np.searchsorted(p, hi, "left")
    return v[a:b].copy(), (p[a:b] - lo).astype(np.int64)


def _slice_runs(v, s, e, lo, hi):
    # runs overlapping [lo, hi): first run whose end >= lo, last whose start < hi;
    # runs crossing a cut are clipped (value duplicated), positions rebased
    a, b = np.searchsorted(e, lo, "left"), np.searchsorted(s, hi, "left")
    ss = np.maximum(s[a:b], lo) - lo
    ee = np.minimum(e[a:b], hi - 1) - lo
    return v[a:b].copy(), ss.astype(np.int64), ee.astype(np.int64)


def shard_column(col, lo: int, hi: int):
    """Rows [lo, hi) of a host column image as a standalone shard (same
    result as the product's rq_shard_host_column; tests/test_oracle_cpu.py
    checks the two agree)."""
    if isinstance(col, H.PlainColumn):
        return H.PlainColumn(col.values[lo:hi].copy(), col.logical, col.center)
    if isinstance(col, H.PlainPlusIndexColumn):
        v, p = _slice_points(col.outliers.v, col.outliers.p, lo, hi)
        return H.PlainPlusIndexColumn(shard_column(col.base, lo, hi), H.IndexColumn(v, p, hi - lo))
    if isinstance(col, H.RleColumn):
        s = col.s if col.s is not None else np.concatenate([[0], col.e[:-1] + 1]).astype(np.int64)
        v, ss, ee = _slice_runs(col.v, s, col.e, lo, hi)
        return H.RleColumn(v, ss, ee, hi - lo)
    if isinstance(col, H.IndexColumn):
        v, p = _slice_points(col.v, col.p, lo, hi)
        return H.IndexColumn(v, p, hi - lo)
    if isinstance(col, H.RlePlusIndexColumn):
        return H.RlePlusIndexColumn(shard_column(col.runs, lo, hi), shard_column(col.points, lo, hi))
    raise TypeError(type(col))


def shard_map(host: dict, nshards: int) -> dict:
    """Every column cut into `nshards` equal row ranges."""
    out = {}
    for k, col in host.items():
        n = col.total_size
        cuts = [n * i // nshards for i in range(nshards + 1)]
        out[k] = [shard_column(col, lo, hi) for lo, hi in zip(cuts[:-1], cuts[1:])]
    return out
