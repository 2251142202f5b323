"""CPU: dictionary codes and literal resolution (dictionary.hpp:16-43,
runner.cpp:106-112, ingest.cpp:72-89)."""
import numpy as np
import pytest

from paper_2506_10092_b200.dictionary import Dictionary, date_literal


def test_first_occurrence_codes():
    d = Dictionary()
    codes = d.encode(["MAIL", "SHIP", "MAIL", "AIR", "SHIP"])
    assert codes.tolist() == [0, 1, 0, 2, 1]
    assert codes.dtype == np.int64
    assert d.size() == 3 and d.at(2) == "AIR" and d.find("SHIP") == 1


def test_literal_absent_is_minus_one():
    d = Dictionary(["A", "N", "R"])
    assert d.literal("N") == 1
    assert d.literal("missing") == -1
    with pytest.raises(ValueError):
        d.at(3)


@pytest.mark.parametrize("tok,days", [("1970-01-01", 0), ("1994-01-01", 8766), ("1998-12-01", 10561),
                                      ("1969-12-31", -1), ("2000-02-29", 11016)])
def test_date_literal(tok, days):
    assert date_literal(tok) == days


@pytest.mark.parametrize("bad", ["1994-1-01", "19940101", "1994-02-30", "abcd-ef-gh"])
def test_date_literal_rejects(bad):
    with pytest.raises(ValueError):
        date_literal(bad)
