"""Summarise `ncu --metrics dram__bytes_*,gpu__time_duration` CSVs of one query
step (tools/traffic.sh) into per-kernel traffic: python tools/traffic_summary.py gpurun_out/traffic_*.csv"""
import csv
import re
import sys
from collections import OrderedDict

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
        "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}


def load(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    k = OrderedDict()
    for r in rows[1:]:
        if not r[ix["ID"]].isdigit():
            continue
        kid = int(r[ix["ID"]])
        name = re.sub(r"\(.*", "", r[ix["Kernel Name"]]).replace("void ", "")
        name = re.sub(r"<.*", "", name).split("::")[-1]
        d = k.setdefault(kid, {"name": name})
        d[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", "")) * UNIT.get(r[ix["Metric Unit"]], 1)
    return k


for p in sys.argv[1:]:
    k = load(p)
    agg = OrderedDict()
    for d in k.values():
        a = agg.setdefault(d["name"], [0, 0.0, 0.0])
        a[0] += 1
        a[1] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
        a[2] += d.get("gpu__time_duration.sum", 0)
    tb = sum(a[1] for a in agg.values())
    tt = sum(a[2] for a in agg.values())
    print(f"== {p}: {len(k)} launches, {tb / 1e9:.3f} GB DRAM, {tt * 1e3:.3f} ms serialised kernel time")
    for n, a in sorted(agg.items(), key=lambda x: -x[1][2])[:12]:
        print(f"  {n:34s} x{a[0]:<4d} {a[1] / 1e6:10.1f} MB {a[2] * 1e3:8.4f} ms  {100 * a[2] / tt:5.1f}%"
              f"  {a[1] / a[2] / 1e9 if a[2] else 0:7.0f} GB/s")
