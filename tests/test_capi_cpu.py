"""CPU: the C-ABI library loads and exports every entry point declared in
include/runq_b200.h (no device compute without a GPU), the ctypes prototype
table matches the header, and the host-only shard slicer behaves."""
import ctypes as C
import os
import re

import numpy as np

from paper_2506_10092_b200 import _lib
from paper_2506_10092_b200 import datagen as G
from paper_2506_10092_b200 import host as H

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "runq_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(rq_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(_lib.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_prototype_table_matches_header():
    assert sorted(_lib.PROTOTYPES) == declared_symbols()


def test_version_and_no_device_error_path():
    lib = _lib.load()
    assert b"sm_100a" in lib.rq_version()
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if not has_gpu:
        h = C.c_void_p()
        st = lib.rq_ctx_create(0, C.byref(h))
        assert st != 0  # fails with a status code, never crashes or falls back
        assert lib.rq_last_error()


def _shard_reference(col, lo, hi):
    pos, vals = H.column_rows(col)
    keep = (pos >= lo) & (pos < hi)
    return pos[keep] - lo, vals[keep]


def test_shard_slicer_rebases_and_splits_runs():
    from paper_2506_10092_b200.runq import shard_host_column
    rng = np.random.default_rng(3)
    for enc in (H.ENC_PLAIN, H.ENC_RLE, H.ENC_INDEX, H.ENC_PLAIN_INDEX, H.ENC_RLE_INDEX):
        col = G.random_column(rng, enc, 1000)
        cuts = [0, 137, 500, 501, 999, 1000]
        total_rows = 0
        for lo, hi in zip(cuts[:-1], cuts[1:]):
            sh = shard_host_column(col, lo, hi)
            assert sh.total_size == hi - lo
            p, v = H.column_rows(sh)
            wp, wv = _shard_reference(col, lo, hi)
            assert np.array_equal(p, wp) and np.array_equal(v, wv), (enc, lo, hi)
            total_rows += len(p)
        assert total_rows == len(H.column_rows(col)[0])


def test_oracle_side_numpy_slicer_matches_product_slicer():
    """bench.py's reference / cpu_baseline legs slice shards with the numpy
    slicer in oracle/refpy.py (they must not load librunq_b200.so); it must
    give exactly the product's rq_shard_host_column shards."""
    from oracle.refpy import shard_column
    from paper_2506_10092_b200.runq import shard_host_column
    rng = np.random.default_rng(4)
    for enc in (H.ENC_PLAIN, H.ENC_RLE, H.ENC_INDEX, H.ENC_PLAIN_INDEX, H.ENC_RLE_INDEX):
        for rep in range(4):
            col = G.random_column(rng, enc, 2000)
            cuts = sorted({0, 2000, *rng.integers(0, 2001, 4).tolist()})
            for lo, hi in zip(cuts[:-1], cuts[1:]):
                a, b = shard_column(col, lo, hi), shard_host_column(col, lo, hi)
                ia, ib = H.column_image(a)[0], H.column_image(b)[0]
                assert type(a) is type(b) and a.total_size == b.total_size
                pa, va = H.column_rows(a)
                pb, vb = H.column_rows(b)
                assert np.array_equal(pa, pb) and np.array_equal(va, vb), (enc, lo, hi)
                assert ia.n == ib.n and ia.n2 == ib.n2, (enc, lo, hi)
