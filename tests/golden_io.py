"""Decoding of tests/golden/fixtures.json into host column images."""
import json
import os

import numpy as np

from paper_2506_10092_b200 import host as H

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "fixtures.json")


def load_cases():
    with open(PATH) as f:
        return json.load(f)["cases"]


def col(d):
    enc = d["enc"]
    if enc == "plain":
        return H.PlainColumn(np.array(d["values"], dtype=H.DTYPES[d["dtype"]]), d["logical"], d["center"])
    if enc == "rle":
        return H.RleColumn(np.array(d["v"], dtype=H.DTYPES[d["dtype"]]), d["s"], d["e"], d["total_size"])
    if enc == "index":
        return H.IndexColumn(np.array(d["v"], dtype=H.DTYPES[d["dtype"]]), d["p"], d["total_size"])
    if enc == "plain+index":
        return H.PlainPlusIndexColumn(col(d["base"]), col(d["outliers"]))
    return H.RlePlusIndexColumn(col(d["runs"]), col(d["points"]))


def mask(d):
    enc = d["enc"]
    if enc == "plain":
        return H.PlainMask(np.array(d["bits"], np.uint8))
    if enc == "rle":
        return H.RleMask(d["s"], d["e"], d["total_size"])
    if enc == "index":
        return H.IndexMask(d["p"], d["total_size"])
    return H.CompositeMask(mask(d["runs"]), mask(d["points"]))


def arr(d):
    return np.array(d["data"], dtype=H.DTYPES[d["dtype"]])


def scal(d):
    return float(d["f64"]) if "f64" in d else int(d["i64"])


def i64(x):
    return np.array(x, dtype=np.int64)
