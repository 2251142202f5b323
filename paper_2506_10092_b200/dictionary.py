"""Dictionary codes for string literals (host side of §8(a) row a20).

Restates ``runq::Dictionary`` (dictionary.hpp:16-43): a bijective
string <-> code table with dense codes in FIRST-OCCURRENCE order, and the
runner's literal resolution (runner.cpp:106-112): a string literal compared
against a dictionary-coded column becomes its code, or −1 when absent (so an
equality never matches). Codes follow first occurrence, so ``<`` on codes is
code order, not string order — exactly as in the reference. The comparison
itself runs on the device (compare_scalar on the int64 code column).
"""
from __future__ import annotations

from typing import Dict, Iterable, List, Optional

import numpy as np


class Dictionary:
    def __init__(self, strings: Iterable[str] = ()):
        self._to_str: List[str] = []
        self._to_code: Dict[str, int] = {}
        for s in strings:
            self.intern(s)

    def intern(self, s: str) -> int:
        code = self._to_code.get(s)
        if code is None:
            code = len(self._to_str)
            self._to_str.append(s)
            self._to_code[s] = code
        return code

    def find(self, s: str) -> Optional[int]:
        return self._to_code.get(s)

    def at(self, code: int) -> str:
        if not 0 <= code < len(self._to_str):
            raise ValueError("dictionary: code out of range")
        return self._to_str[code]

    def size(self) -> int:
        return len(self._to_str)

    def encode(self, values: Iterable[str]) -> np.ndarray:
        """Interns every value (ingest order) and returns int64 codes."""
        return np.fromiter((self.intern(v) for v in values), dtype=np.int64)

    def literal(self, s: str) -> int:
        """runner.cpp:106-112: the code of a string literal, −1 if absent."""
        code = self.find(s)
        return -1 if code is None else code


def date_literal(tok: str) -> int:
    """parse_date_literal (ingest.cpp:72-89): 'YYYY-MM-DD' -> days since
    1970-01-01 (proleptic Gregorian); malformed dates raise."""
    import datetime
    if len(tok) != 10 or tok[4] != "-" or tok[7] != "-":
        raise ValueError(f"not a date (YYYY-MM-DD): '{tok}'")
    d = datetime.date(int(tok[0:4]), int(tok[5:7]), int(tok[8:10]))
    return (d - datetime.date(1970, 1, 1)).days
