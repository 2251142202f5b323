"""GPU parity: column images (rq_col_dump_image / rq_col_load_image) against
the reference's dump_column (column.cpp:513-563) — byte-identical images for
every encoding, storage width, centre and float value type, and the image
loaded back to the device round-trips to the same column (the reference's
test_column.cpp:115-141 checks, header fields and body = stats bytes)."""
import json

import numpy as np
import pytest

from helpers import assert_column
from paper_2506_10092_b200 import datagen as G
from paper_2506_10092_b200 import host as H
from paper_2506_10092_b200._lib import RqError

pytestmark = pytest.mark.gpu
ENCS = [H.ENC_PLAIN, H.ENC_RLE, H.ENC_INDEX, H.ENC_PLAIN_INDEX, H.ENC_RLE_INDEX]
ENC_NAMES = ["plain", "rle", "index", "plain+index", "rle+index"]


def _split(img: bytes):
    nl = img.index(b"\n")
    return json.loads(img[:nl].decode()), img[nl + 1:]


@pytest.mark.parametrize("enc", range(5), ids=lambda e: ENC_NAMES[e])
@pytest.mark.parametrize("flt", [False, True], ids=["int", "float"])
def test_dump_matches_reference_bytes(rq, ref, enc, flt):
    rng = np.random.default_rng(300 + 2 * enc + flt)
    for inst in range(5):
        n = int(rng.integers(1, 3000))
        c = G.random_column(rng, ENCS[enc], n, flt, True, 40)
        got = rq.dump_image(c)
        want = ref.dump_column(c)
        assert got == want, f"{ENC_NAMES[enc]} inst {inst}: header {got[:120]!r} vs {want[:120]!r}"
        back = rq.load_image(want).download()
        assert_column(back, c, f"load {ENC_NAMES[enc]} inst {inst}")


def test_reference_dump_example(rq, ref):
    # test_column.cpp:115-129: the worked example's header and body length
    c = H.RleColumn(v=np.array([5, 6], dtype=np.int32), s=np.array([0, 4]), e=np.array([1, 6]), total_size=8)
    img = rq.dump_image(c)
    assert img == ref.dump_column(c)
    hdr, body = _split(img)
    assert hdr["encoding"] == "rle" and hdr["total_size"] == 8
    assert hdr["widths"] == {"value": 4, "position": 8}
    assert len(body) == 2 * (4 + 16)


@pytest.mark.parametrize("dt,name", [(np.int8, "i8"), (np.int16, "i16"), (np.int32, "i32")], ids=["i8", "i16", "i32"])
def test_narrow_plain_storage_and_centre(rq, ref, dt, name):
    rng = np.random.default_rng(7)
    v = rng.integers(-100, 100, 1000).astype(dt)
    for center in (None, 0, 12345):
        c = H.PlainColumn(values=v, logical=H.I64, center=center)
        img = rq.dump_image(c)
        assert img == ref.dump_column(c)
        hdr, _ = _split(img)
        assert hdr["storage"] == name and hdr["value_type"] == "i64"
        assert ("center" in hdr) == (center is not None)
        assert_column(rq.load_image(img).download(), c, f"plain {dt} centre {center}")


def test_empty_columns(rq, ref):
    for c in (H.RleColumn(v=np.zeros(0, np.int64), s=np.zeros(0, np.int64), e=np.zeros(0, np.int64), total_size=10),
              H.IndexColumn(v=np.zeros(0, np.float64), p=np.zeros(0, np.int64), total_size=5)):
        img = rq.dump_image(c)
        assert img == ref.dump_column(c)
        assert_column(rq.load_image(img).download(), c, "empty")


def test_malformed_images_raise(rq, ref):
    c = H.RleColumn(v=np.array([1, 2], dtype=np.int64), s=np.array([0, 5]), e=np.array([4, 9]), total_size=10)
    img = ref.dump_column(c)
    with pytest.raises(RqError):
        rq.load_image(img[:-1])  # truncated body
    with pytest.raises(RqError):
        rq.load_image(img + b"\x00")  # trailing bytes
    with pytest.raises(RqError):
        rq.load_image(img.replace(b'"rle"', b'"xyz"'))
    with pytest.raises(RqError):
        rq.load_image(b"no header line")
