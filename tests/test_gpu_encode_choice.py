"""GPU: the synthetic lineitem's encodings are the ones the ingest heuristic
picks (choose_encoding, ingest.cpp:217-271 — the device implementation,
checked against the reference's in tests/test_gpu_encode.py): every column of
the SF100 Q1 and Q6 tables is decoded on the device (decode_full) and
re-chosen from its 600M logical values (VERDICT r1 "measurement gaps": build
the C4 columns by the heuristic instead of asserting it)."""
import pytest

from paper_2506_10092_b200 import host as H
from paper_2506_10092_b200 import queries as Q

pytestmark = pytest.mark.gpu

SF100 = 600_000_000


def _chosen(rq, col):
    d = rq.upload(col)
    values = rq.decode_full(d)
    plain = rq.make_plain(values)
    return rq.io.choose_encoding(plain)


def _check(rq, t):
    for name, col in t.items():
        ch = _chosen(rq, col)
        if isinstance(col, H.RleColumn):
            assert ch.scheme == H.SCHEME_RLE, (name, ch.as_tuple())
        else:
            assert isinstance(col, H.PlainColumn)
            if col.values.dtype.kind == "f":
                assert ch.scheme == H.SCHEME_PLAIN and ch.width == H.F64, (name, ch.as_tuple())
            else:  # plain-centered at the generator's width and centre
                assert ch.scheme == H.SCHEME_PLAIN_CENTERED, (name, ch.as_tuple())
                assert ch.width == H.dtype_code(col.values) and ch.center == col.center, (name, ch.as_tuple())


def test_q1_sf100_encodings_are_the_heuristics(rq):
    _check(rq, Q.lineitem_q1(SF100, 43))


def test_q6_sf100_encodings_are_the_heuristics(rq):
    _check(rq, Q.lineitem_q6(SF100, 42))
