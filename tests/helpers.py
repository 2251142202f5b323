"""Structural comparison helpers: parity means the SAME encoding, the same
dtypes and the same arrays (bit-exact for positions, masks, counts and
integers; |x-y| <= 1e-9*max(1,|x|,|y|) for f64, runner.cpp:394-402 /
oracle.hpp:258-261)."""
import numpy as np

from paper_2506_10092_b200 import host as H

REL = 1e-9


def approx_equal(a, b, rel=REL):
    a = np.asarray(a)
    b = np.asarray(b)
    if a.shape != b.shape:
        return False
    if a.dtype.kind == "f" or b.dtype.kind == "f":
        a = a.astype(np.float64)
        b = b.astype(np.float64)
        both_nan = np.isnan(a) & np.isnan(b)
        tol = rel * np.maximum(1.0, np.maximum(np.abs(a), np.abs(b)))
        ok = both_nan | (np.abs(a - b) <= tol) | (a == b)
        return bool(ok.all())
    return bool(np.array_equal(a, b))


def assert_array(got, want, what="", exact_dtype=True):
    got = np.asarray(got)
    want = np.asarray(want)
    if exact_dtype:
        assert got.dtype == want.dtype, f"{what}: dtype {got.dtype} != {want.dtype}"
    assert got.shape == want.shape, f"{what}: shape {got.shape} != {want.shape}"
    assert approx_equal(got, want), f"{what}: values differ\n got={got[:20]}\nwant={want[:20]}"


def assert_column(got, want, what=""):
    assert type(got) is type(want), f"{what}: encoding {type(got).__name__} != {type(want).__name__}"
    assert got.total_size == want.total_size, f"{what}: total_size {got.total_size} != {want.total_size}"
    if isinstance(want, H.PlainColumn):
        assert got.logical == want.logical, f"{what}: logical dtype"
        assert got.center == want.center, f"{what}: center"
        assert_array(got.values, want.values, what + ".values")
    elif isinstance(want, H.RleColumn):
        assert_array(got.s, want.s, what + ".s")
        assert_array(got.e, want.e, what + ".e")
        assert_array(got.v, want.v, what + ".v")
    elif isinstance(want, H.IndexColumn):
        assert_array(got.p, want.p, what + ".p")
        assert_array(got.v, want.v, what + ".v")
    elif isinstance(want, H.PlainPlusIndexColumn):
        assert_column(got.base, want.base, what + ".base")
        assert_array(got.outliers.p, want.outliers.p, what + ".outliers.p")
        assert_array(got.outliers.v, want.outliers.v, what + ".outliers.v")
    else:
        assert_column(got.runs, want.runs, what + ".runs")
        assert_array(got.points.p, want.points.p, what + ".points.p")
        assert_array(got.points.v, want.points.v, what + ".points.v")


def assert_mask(got, want, what=""):
    assert type(got) is type(want), f"{what}: mask encoding {type(got).__name__} != {type(want).__name__}"
    assert got.total_size == want.total_size, f"{what}: total_size"
    if isinstance(want, H.PlainMask):
        assert_array(got.bits != 0, want.bits != 0, what + ".bits", exact_dtype=False)
    elif isinstance(want, H.RleMask):
        assert_array(got.s, want.s, what + ".s")
        assert_array(got.e, want.e, what + ".e")
    elif isinstance(want, H.IndexMask):
        assert_array(got.p, want.p, what + ".p")
    else:
        assert_array(got.runs.s, want.runs.s, what + ".runs.s")
        assert_array(got.runs.e, want.runs.e, what + ".runs.e")
        assert_array(got.points.p, want.points.p, what + ".points.p")


def assert_scalar(got, want, what=""):
    if isinstance(want, float):
        assert isinstance(got, float), f"{what}: expected f64 result, got {type(got)}"
        assert approx_equal(np.array([got]), np.array([want])), f"{what}: {got} != {want}"
    else:
        assert isinstance(got, int), f"{what}: expected i64 result, got {type(got)}"
        assert got == want, f"{what}: {got} != {want}"
