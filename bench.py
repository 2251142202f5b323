#!/usr/bin/env python
"""Benchmark of the compressed-execution query path (BASELINE.json metric:
logical rows/s per query and % of HBM roofline on compressed bytes).

Default workload = BASELINE config[1] (C2): filtered SUM(A*B) WHERE C < k
over 1B logical rows per GPU — A RLE int64 (L=64, 15.6M runs), B Index int64
(1% density, 10M points), C dictionary codes (cardinality 64) RLE L=256.
A step is one execution of the query through the C ABI on device-resident
compressed columns (`value`); `e2e` repeats it through the same call with
the compressed columns uploaded from pinned host memory every step and the
result read back. Inputs exceed L2 (126 MB), so no flush is needed.

Other workloads (--workload): c1 = SUM(A+B) over two misaligned RLE int64
columns (fused rq_aggregate_binop), c3 = GROUP BY dict key SUM/COUNT/AVG over
RLE / RLE+Index / bit-width-reduced i16 / f64 columns (fused group-by).

Multi-GPU (torchrun): one process per GPU, each rank owns a row-range shard
of the same size (weak scaling); the per-rank partial aggregate is merged
with one NCCL all_reduce per step.

--impl reference runs the UNMODIFIED reference library (oracle/_ref, the
reference compiled from its sources) on the same workload on the host's
cores (row-range shards on all threads; the reference is single-threaded),
rank 0 only.
"""
import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "logical rows/s per query and % HBM roofline on compressed bytes, 1/2/4/8 B200"
UNIT = "rows/s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """NVML sampling of SM clock + throttle reasons during the timed region."""

    REASONS = {
        0x0000000000000008: "hw_slowdown",
        0x0000000000000040: "hw_thermal_slowdown",
        0x0000000000000020: "sw_thermal_slowdown",
        0x0000000000000004: "sw_power_cap",
    }

    def __init__(self, device):
        self.samples, self.reasons = [], set()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as ex:  # pragma: no cover
            log("nvml unavailable:", ex)
        self._stop = threading.Event()

    def _sample(self):
        nv = self.nv
        self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        for bit, name in self.REASONS.items():
            if r & bit:
                self.reasons.add(name)

    def _run(self):
        # every 10 ms: NVML queries take driver locks that delay the launches
        # and syncs of host-paced steps (Q6 / C5: 27 launches per 0.4 ms step)
        while not self._stop.is_set():
            self._sample()
            self._stop.wait(0.01)

    def __enter__(self):
        if self.ok:
            self._sample()
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()
            self._sample()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml-unavailable"]}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": float(self.max),
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


_PINNED = []  # keeps pinned host tensors alive


def pinned_copy(a: np.ndarray) -> np.ndarray:
    import torch
    t = torch.empty(max(1, a.nbytes), dtype=torch.uint8, pin_memory=True)
    _PINNED.append(t)
    out = t.numpy().view(a.dtype)[: a.shape[0]]
    out[:] = a
    return out


def pin_column(col):
    from paper_2506_10092_b200 import host as H
    if isinstance(col, H.RleColumn):
        # gapless columns cross PCIe without their (implied) starts
        s = None if col.is_gapless() else pinned_copy(col.s)
        return H.RleColumn(pinned_copy(col.v), s, pinned_copy(col.e), col.total_size)
    if isinstance(col, H.IndexColumn):
        return H.IndexColumn(pinned_copy(col.v), pinned_copy(col.p), col.total_size)
    if isinstance(col, H.PlainColumn):
        return H.PlainColumn(pinned_copy(col.values), col.logical, col.center)
    if isinstance(col, H.RlePlusIndexColumn):
        return H.RlePlusIndexColumn(pin_column(col.runs), pin_column(col.points))
    if isinstance(col, H.PlainPlusIndexColumn):
        return H.PlainPlusIndexColumn(pin_column(col.base), pin_column(col.outliers))
    raise TypeError(type(col))


def col_bytes(col):
    from paper_2506_10092_b200 import host as H
    if isinstance(col, H.RleColumn):
        return col.v.nbytes + (col.s.nbytes if col.s is not None else 0) + col.e.nbytes
    if isinstance(col, H.IndexColumn):
        return col.v.nbytes + col.p.nbytes
    if isinstance(col, H.RlePlusIndexColumn):
        return col_bytes(col.runs) + col_bytes(col.points)
    if isinstance(col, H.PlainPlusIndexColumn):
        return col_bytes(col.base) + col_bytes(col.outliers)
    return col.values.nbytes


def alg_bytes(col, gapless=True, only_points=None):
    """ALG_BYTES per SURVEY.md §8d: gapless RLE R·(w_v+8) (v + e; s implied),
    gapped RLE R·(w_v+16), Index P·(w_v+8), Plain n·w_storage (or P·w when
    read only at P positions), composites = sum of parts."""
    from paper_2506_10092_b200 import host as H
    if isinstance(col, H.RleColumn):
        return col.v.shape[0] * (col.v.itemsize + (8 if gapless else 16))
    if isinstance(col, H.IndexColumn):
        return col.p.shape[0] * (col.v.itemsize + 8)
    if isinstance(col, H.RlePlusIndexColumn):
        return alg_bytes(col.runs, gapless=False) + alg_bytes(col.points)
    n = only_points if only_points is not None else col.values.shape[0]
    return n * col.values.itemsize


def ncu_traffic(workload, tag):
    """dram bytes per launch of the dominant kernel (tag) or of the whole
    query step (tag "query") of one workload, from the committed ncu captures
    (profiles/ncu_traffic.json, keyed "<workload>:<tag>"), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(f"{workload}:{tag}", {}).get("dram_bytes_per_launch")
    except Exception:
        return None


# ---------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------


class C2:
    name = "c2"
    tag = "filtered_points_reduce"
    dtype = "int64"

    def __init__(self, args):
        self.args = args
        self.k = 20

    def describe(self):
        cdesc = "RLE L=256" if self.args.variant == "rle" else "plain-centered i8 L=4"
        return (f"C2: filtered SUM(A*B) WHERE C<{self.k}; A RLE i64 L=64, B Index i64 1%, "
                f"C dict codes (card 64) {cdesc}")

    def gen(self, rows, seed):
        from paper_2506_10092_b200 import datagen as G
        a, b, c = G.c2_tables(rows, seed=seed, c_variant=self.args.variant)
        self.host = {"a": a, "b": b, "c": c}
        return self.host

    def alg_bytes(self, h):
        from paper_2506_10092_b200 import host as H
        c = h["c"]
        cb = alg_bytes(c) if isinstance(c, H.RleColumn) else alg_bytes(c, only_points=h["b"].p.shape[0])
        return alg_bytes(h["a"]) + alg_bytes(h["b"]) + cb

    def query(self, rq, d, path):
        if path == "fused":
            return rq.agg.filtered_aggregate_binop(d["c"], self.k, "<", d["a"], d["b"], "*", "sum")
        m = rq.compute.compare_scalar(d["c"], self.k, "<")
        return rq.agg.aggregate_all(rq.compute.arith(rq.compute.filter(d["a"], m), rq.compute.filter(d["b"], m), "*"),
                                    "sum")

    def oracle(self, h):
        from oracle import refpy
        return refpy.Orq().filtered_sum(h["c"], self.k, "<", h["a"], h["b"], "*")

    def ref_run(self, ref, shards, threads):
        return ref.chain_filtered_sum(shards["c"], shards["a"], shards["b"], threads, self.k, "<", "*")


class C1:
    name = "c1"
    tag = "pair_reduce"
    dtype = "int64"

    def __init__(self, args):
        self.args = args

    def describe(self):
        return "C1: SUM(A+B) over two misaligned RLE i64 columns, L=64/96"

    def gen(self, rows, seed):
        from paper_2506_10092_b200 import datagen as G
        a, b = G.c1_tables(rows, 64, 96, seed)
        self.host = {"a": a, "b": b}
        return self.host

    def alg_bytes(self, h):
        return alg_bytes(h["a"]) + alg_bytes(h["b"])

    def query(self, rq, d, path):
        if path == "fused":
            return rq.agg.aggregate_binop(d["a"], d["b"], "+", "sum")
        return rq.agg.aggregate_all(rq.compute.arith(d["a"], d["b"], "+"), "sum")

    def oracle(self, h):
        from oracle import refpy
        return refpy.Orq().sum_rle_binop(h["a"], h["b"], "+")

    def ref_run(self, ref, shards, threads):
        return ref.chain_sum_binop(shards["a"], shards["b"], threads, "+")


def table_summary(t):
    """JSON-friendly digest of a group table (keys, values): group count and
    per-column sums."""
    keys, vals = t
    return {"groups": int(len(keys[0])) if keys else 1,
            "column_sums": [int(np.asarray(v).astype(np.int64).sum()) if np.asarray(v).dtype.kind != "f"
                            else float(np.nansum(v)) for v in vals]}


def tables_same(a, b):
    """Group tables equal: keys / ints bit-exact, f64 within 1e-9 relative,
    NaN == NaN (runner.cpp:394-402)."""
    (ka, va), (kb, vb) = a, b
    if len(ka) != len(kb) or len(va) != len(vb):
        return False
    for x, y in zip(ka, kb):
        if not np.array_equal(np.asarray(x).astype(np.int64), np.asarray(y).astype(np.int64)):
            return False
    for x, y in zip(va, vb):
        x, y = np.asarray(x), np.asarray(y)
        if x.shape != y.shape:
            return False
        if x.dtype.kind == "f" or y.dtype.kind == "f":
            x, y = x.astype(np.float64), y.astype(np.float64)
            tol = 1e-9 * np.maximum(1.0, np.maximum(np.abs(x), np.abs(y)))
            if not np.all((np.isnan(x) & np.isnan(y)) | (np.abs(x - y) <= tol)):
                return False
        elif not np.array_equal(x.astype(np.int64), y.astype(np.int64)):
            return False
    return True


class C3:
    name = "c3"
    tag = "group_fused"
    dtype = "int64/f64"
    host_rows_max = 2_000_000_000  # above this Z / W stream into HBM chunk by chunk (never whole on the host)
    same = staticmethod(tables_same)
    summary = staticmethod(table_summary)

    def __init__(self, args):
        self.args = args
        self.fold = None

    def describe(self):
        return ("C3: GROUP BY K (codes 0..99, RLE L=4096) -> SUM(X RLE L=128), COUNT(*), AVG(Z plain-centered i16), "
                "SUM(Y RLE+Index 90% runs L=256 / 10% points), SUM(W plain f64)")

    def gen(self, rows, seed):
        from paper_2506_10092_b200 import datagen as G
        self.rows, self.seed = rows, seed
        self.chunked = rows > self.host_rows_max
        if self.chunked:
            k, x, y = G.c3_run_columns(rows, seed)
            self.host = {"k": k, "x": x, "y": y}
        else:
            k, x, y, z, w = G.c3_tables(rows, seed)
            self.host = {"k": k, "x": x, "y": y, "z": z, "w": w}
        return self.host

    def upload(self, rq, ctx, host, check):
        """Chunked tables: Z / W generated chunk by chunk, written into HBM
        (rq_arr_alloc + rq_arr_write) and, when `check`, folded into the
        streaming oracle as they pass."""
        dev = {k: rq.upload(v, ctx) for k, v in host.items()}
        if not self.chunked:
            return dev
        from paper_2506_10092_b200 import datagen as G
        from paper_2506_10092_b200 import host as H
        if check:
            from oracle import streaming as S
            self.fold = S.C3Fold(S.StreamingOracle(), host["k"], host["x"], host["y"])
        za, wa = rq.alloc_array(H.I16, self.rows, ctx), rq.alloc_array(H.F64, self.rows, ctx)
        t0 = time.time()
        for r0 in range(0, self.rows, G.C3_CHUNK):
            z, w = G.c3_plain_chunk(self.rows, self.seed, r0)
            keep = (za.write(r0, z), wa.write(r0, w))
            if self.fold is not None:
                self.fold.add_plain_chunk(r0, H.PlainColumn(z, H.I64, 0), w)
            ctx.synchronize()
            del keep
        log(f"streamed Z/W ({self.rows} rows) into HBM in {time.time() - t0:.1f}s")
        dev["z"], dev["w"] = rq.make_plain(za, H.I64, 0), rq.make_plain(wa)
        return dev

    def alg_bytes(self, h):
        b = sum(alg_bytes(h[n]) for n in ("k", "x", "y"))
        return b + self.rows * (2 + 8)  # Z i16 + W f64 per row

    def query(self, rq, d, path):
        from paper_2506_10092_b200 import datagen as G
        ks, vs, ng = rq.agg.group_aggregate([d["k"]], [d["x"], d["k"], d["z"], d["y"], d["w"]], G.C3_FNS,
                                            normalize=True)
        h = rq.download_all(list(ks) + list(vs))
        return h[:1], h[1:]

    def oracle(self, h):
        """The full group table from the streaming oracle (oracle/streaming.py,
        pinned against the reference library up to 100M rows)."""
        if self.fold is not None:
            return self.fold.result()
        from oracle import streaming as S
        return S.c3(h)

    def cpu_sample(self, host, rows):
        if not self.chunked:
            return None
        from paper_2506_10092_b200 import datagen as G
        k, x, y, z, w = G.c3_tables(rows, self.seed)
        return {"k": k, "x": x, "y": y, "z": z, "w": w}

    def ref_run(self, ref, shards, threads):
        from paper_2506_10092_b200 import datagen as G
        t0 = time.perf_counter()
        tot = 0
        for i in range(len(shards["k"])):
            kk = ref.normalize_basic(shards["k"][i])
            cols = [ref.normalize_basic(shards[n][i]) for n in ("x", "k", "z", "y", "w")]
            ks, vs, ng = ref.group_aggregate([kk], cols, G.C3_FNS)
            tot += int(vs[0].astype(np.int64).sum())
        return tot, time.perf_counter() - t0


class Q6:
    """C4: TPC-H-style Q6 over synthetic lineitem (SF = rows / 6M) sorted by
    (quantity, discount, shipdate) — device operator chain, same plan as the
    reference runner."""
    name = "q6"
    tag = None  # whole query (operator chain)
    dtype = "f64"
    ref_rows = 60_000_000  # reference arm sample (SF10)

    def __init__(self, args):
        self.args = args
        # fused path: the K12 row kernel (the query's dominant kernel); chain: whole query
        self.tag = "xg_rows" if args.path == "fused" else None

    def describe(self):
        return (f"C4 Q6: SUM(price*disc) WHERE shipdate in [1994-01-01,1995-01-01) AND disc BETWEEN 5 AND 7 AND "
                f"qty < 24; lineitem SF{self.args.rows / 6e6:g} sorted (qty, disc, shipdate), RLE keys + f64 price")

    def gen(self, rows, seed):
        from paper_2506_10092_b200 import queries as Q
        self.host = Q.lineitem_q6(rows, seed)
        return self.host

    def alg_bytes(self, h):
        from paper_2506_10092_b200 import queries as Q
        sd, d, q = h["l_shipdate"], h["l_discount"], h["l_quantity"]
        # price is read only at the selected rows: estimate them from the runs
        sel = self._selected(h)
        if self.tag == "xg_rows":  # the row kernel reads price at the selected rows
            return sel * 8
        return alg_bytes(sd) + alg_bytes(d) + alg_bytes(q) + sel * 8

    def _selected(self, h):
        from paper_2506_10092_b200 import queries as Q
        sd, d, q = h["l_shipdate"], h["l_discount"], h["l_quantity"]
        # runs of shipdate inside a passing (qty, disc) block and date range
        qi = np.searchsorted(q.e, sd.s)
        di = np.searchsorted(d.e, sd.s)
        ok = (q.v[qi] < 24) & (d.v[di] >= 5) & (d.v[di] <= 7) & (sd.v >= Q.Q6_LO) & (sd.v < Q.Q6_HI)
        return int((sd.e - sd.s + 1)[ok].sum())

    def query(self, rq, d, path):
        from paper_2506_10092_b200 import queries as Q
        if path == "fused":
            v, fused = Q.q6_fused(rq, d)
            assert fused, "q6: fused path not taken"
            return v
        return Q.q6(rq, d)

    def oracle(self, h):
        """Streaming oracle (oracle/streaming.py) on the full table."""
        from oracle import streaming as S
        from paper_2506_10092_b200 import queries as Q
        return S.q6(h, Q.Q6_WHERE)

    @staticmethod
    def same(a, b):
        return abs(a - b) <= 1e-9 * max(1.0, abs(a), abs(b))

    def ref_run(self, ref, shards, threads):
        from oracle.refpy import RefAPI
        from paper_2506_10092_b200 import queries as Q
        api = RefAPI(ref)
        t0 = time.perf_counter()
        tot = sum(Q.q6(api, {k: v[i] for k, v in shards.items()}) for i in range(len(shards["l_shipdate"])))
        return tot, time.perf_counter() - t0


class Q1(Q6):
    name = "q1"
    dtype = "int64/f64"
    ref_rows = 2_000_000

    def describe(self):
        return (f"C4 Q1: GROUP BY returnflag, linestatus: 4 SUMs, 3 AVGs, COUNT WHERE shipdate <= 1998-09-02; "
                f"lineitem SF{self.args.rows / 6e6:g} sorted (rf, ls, shipdate, qty); disc/tax i8 plain, price f64")

    def gen(self, rows, seed):
        from paper_2506_10092_b200 import queries as Q
        self.host = Q.lineitem_q1(rows, seed)
        return self.host

    def alg_bytes(self, h):
        if self.tag == "xg_rows":  # the row kernel streams price / disc / tax over the rows passing the filter
            from paper_2506_10092_b200 import queries as Q
            sd = h["l_shipdate"]
            sel = int((sd.e - sd.s + 1)[sd.v <= Q.Q1_CUTOFF].sum())
            return sel * (8 + 1 + 1)
        return sum(alg_bytes(c, gapless=True) for c in h.values())

    def query(self, rq, d, path):
        from paper_2506_10092_b200 import queries as Q
        if path == "fused":
            (ks, vs, ng), fused = Q.q1_fused(rq, d)
            assert fused, "q1: fused path not taken"
        else:
            ks, vs, ng = Q.q1(rq, d)
        h = rq.download_all(list(ks) + list(vs))
        return h[:2], h[2:]

    def oracle(self, h):
        from oracle import streaming as S
        from paper_2506_10092_b200 import queries as Q
        return S.q1(h, Q.Q1_CUTOFF)

    same = staticmethod(tables_same)
    summary = staticmethod(table_summary)

    def ref_run(self, ref, shards, threads):
        from oracle.refpy import RefAPI
        from paper_2506_10092_b200 import queries as Q
        api = RefAPI(ref)
        t0 = time.perf_counter()
        tot = 0
        for i in range(len(shards["l_shipdate"])):
            ks, vs, ng = Q.q1(api, {k: v[i] for k, v in shards.items()})
            tot += int(vs[7].sum())
        return tot, time.perf_counter() - t0


class C5(Q6):
    """C5: production-shaped 15-column table (7 RLE code columns incl. the
    avg-34.41 heavy one, 4 Plain+Index i16+1% outliers, 4 narrow plain);
    WHERE r2 IN (3,17,42) AND r3 < 50 GROUP BY r4: SUM(pi0), SUM(p1), COUNT.
    6B rows over 8 GPUs = 750M rows per GPU (weak scaling per rank)."""
    name = "c5"
    dtype = "int64"
    same = staticmethod(tables_same)
    summary = staticmethod(table_summary)
    ref_rows = 20_000_000
    columns = ["r2", "r3", "r4", "pi0", "p1"]

    def describe(self):
        return ("C5: production-shaped 15 cols (7 RLE i32 codes, 4 Plain+Index i16+1% i64, 4 narrow plain); "
                "WHERE r2 IN (3,17,42) AND r3 < 50 GROUP BY r4 -> SUM(pi0), SUM(p1), COUNT(*)")

    def gen(self, rows, seed):
        from paper_2506_10092_b200 import queries as Q
        self.host = Q.production_table(rows, seed)
        return self.host

    def alg_bytes(self, h):
        # predicate / key runs + the two measures read only at the selected rows
        sel = getattr(self, "_sel", 0)
        runs = sum(alg_bytes(h[k]) for k in ("r2", "r3", "r4"))
        pi0 = h["pi0"]
        if self.tag == "xg_rows":  # the row kernel reads the two i16 measures at the selected rows
            return sel * (2 + 2)
        out_frac = len(pi0.outliers.p) / max(1, pi0.base.values.shape[0])
        return runs + sel * (2 + 2) + int(sel * out_frac) * 16

    def query(self, rq, d, path):
        from paper_2506_10092_b200 import queries as Q
        if path == "fused":
            (ks, vs, ng), fused = Q.c5_fused(rq, d)
            assert fused, "c5: fused path not taken"
        else:
            ks, vs, ng = Q.c5_query(rq, d)
        h = rq.download_all(list(ks) + list(vs))
        self._sel = int(h[3].sum())
        return h[:1], h[1:]

    def oracle(self, h):
        from oracle import streaming as S
        from paper_2506_10092_b200 import queries as Q
        return S.c5(h, Q.C5_IN, Q.C5_LT)

    def ref_run(self, ref, shards, threads):
        from oracle.refpy import RefAPI
        from paper_2506_10092_b200 import queries as Q
        api = RefAPI(ref)
        t0 = time.perf_counter()
        tot = 0
        for i in range(len(shards["r4"])):
            ks, vs, ng = Q.c5_query(api, {k: v[i] for k, v in shards.items()})
            tot += int(vs[2].sum())
        return tot, time.perf_counter() - t0


WORKLOADS = {"c1": C1, "c2": C2, "c3": C3, "q6": Q6, "q1": Q1, "c5": C5}


def shard_map(host, nshards):
    # numpy slicer from the oracle side: the reference / cpu_baseline legs
    # never load the product library
    from oracle.refpy import shard_map as np_shard_map
    return np_shard_map(host, nshards)


def result_bytes(v):
    """Bytes the step reads back: the scalar, or every key / value array of
    a group table."""
    if isinstance(v, tuple) and len(v) == 2 and isinstance(v[0], list):
        return int(sum(np.asarray(a).nbytes for a in v[0] + v[1]))
    return 8


def config_dict(args, w, rows):
    return {"workload": w.describe(), "rows_per_gpu": rows, "query_path": args.path,
            "l2_policy": "inputs larger than L2 (126 MB) - no flush needed"}


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------


def run_reference(args, w, rank, world):
    if rank != 0:
        return
    from oracle import refpy
    ref = refpy.Ref()
    threads = os.cpu_count() or 1
    rows = min(args.rows, getattr(w, "ref_rows", args.rows)) if w.name != "c3" else min(args.rows, 20_000_000)
    host = w.gen(rows, 42)
    nshards = threads if w.name in ("c1", "c2") else 1
    shards = shard_map(host, nshards)
    for _ in range(args.warmup):
        w.ref_run(ref, shards, threads)
    times = []
    val = None
    for _ in range(args.steps):
        val, sec = w.ref_run(ref, shards, threads)
        times.append(sec)
    ms = 1000.0 * statistics.median(times)
    value = rows / (ms / 1000.0)
    cores = threads if nshards > 1 else 1
    # this arm runs only the reference library: the product must not be mapped
    with open("/proc/self/maps") as f:
        product_loaded = "librunq_b200" in f.read()
    assert not product_loaded, "reference arm loaded the product library"
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": w.dtype,
        "data": "synthetic", "config": config_dict(args, w, rows), "result": val,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": f"{rows}-row table as {nshards} row-range shard(s) on {cores} thread(s); "
                                   "the reference operator chain per shard (oracle/_ref)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "product_library_loaded": product_loaded,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--rows", type=int, default=None,
                    help="logical rows per GPU (default 1B; SF100 = 600M for q6/q1)")
    ap.add_argument("--variant", default="rle", choices=["rle", "narrow"])
    ap.add_argument("--path", default="fused", choices=["fused", "chain"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.rows is None:
        args.rows = {"q6": 600_000_000, "q1": 600_000_000, "c5": 750_000_000}.get(args.workload, 1_000_000_000)
    w = WORKLOADS[args.workload](args)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        if args.impl == "ours":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")

    if args.impl == "reference":
        run_reference(args, w, rank, world)
        if dist is not None:
            dist.destroy_process_group()
        return

    import torch
    from paper_2506_10092_b200 import runq

    rows = args.rows
    t0 = time.time()
    host = w.gen(rows, 42 + rank)
    log(f"[rank {rank}] generated {w.name} with {rows} rows in {time.time() - t0:.1f}s")

    ctx = runq.Context(local)
    stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", local))
    check = rank == 0 and world == 1
    if hasattr(w, "upload"):
        dev = w.upload(runq, ctx, host, check)
    else:
        dev = {k: runq.upload(v, ctx) for k, v in host.items()}
    pending = []  # in-flight partial merges (async NCCL all_reduce; completed by the closing barrier)

    def step(d, path=None, merge_async=False):
        v = w.query(runq, d, path or args.path)
        if dist is not None and merge_async:
            # the merge of step i overlaps step i+1's kernels: enqueue the
            # all_reduce of this step's partials and keep the handles alive
            parts = list(v) if isinstance(v, tuple) else [v]
            ints = [x for x in parts if isinstance(x, int)]
            flts = [x for x in parts if not isinstance(x, int)]
            for vals, dt in ((ints, torch.int64), (flts, torch.float64)):
                if vals:
                    t = torch.tensor(vals, dtype=dt, device=f"cuda:{local}")
                    pending.append((t, dist.all_reduce(t, async_op=True)))
            return v
        if dist is not None:
            # partial-aggregate merge over NCCL: every component of the rank's
            # result is a SUM / COUNT partial (int64 wraps like the reference,
            # f64 sums reassociate within tolerance); one all_reduce per dtype
            parts = list(v) if isinstance(v, tuple) else [v]
            ints = [x for x in parts if isinstance(x, int)]
            flts = [x for x in parts if not isinstance(x, int)]
            out_i, out_f = [], []
            if ints:
                ti = torch.tensor(ints, dtype=torch.int64, device=f"cuda:{local}")
                dist.all_reduce(ti)
                out_i = ti.tolist()
            if flts:
                tf = torch.tensor(flts, dtype=torch.float64, device=f"cuda:{local}")
                dist.all_reduce(tf)
                out_f = tf.tolist()
            merged = [out_i.pop(0) if isinstance(x, int) else out_f.pop(0) for x in parts]
            v = tuple(merged) if isinstance(v, tuple) else merged[0]
        return v

    # correctness gate (rank 0, N=1): fused == device chain == oracle. The
    # oracle is the C restatement (C1 / C2) or the streaming group-by oracle
    # (C3 / Q1 / Q6 / C5, oracle/streaming.py) over the FULL table, pinned
    # against the reference library up to 100M rows.
    same = getattr(w, "same", lambda a, b: a == b)
    v_fused = w.query(runq, dev, args.path)
    if args.path == "fused":  # fused kernels == the device operator chain (itself checked vs the reference)
        v_chain = w.query(runq, dev, "chain")
        assert same(v_fused, v_chain), (v_fused, v_chain)
    oracle_ok = None
    if check:
        t1 = time.time()
        want = w.oracle(host)
        if want is not None:
            oracle_ok = bool(same(v_fused, want))
            log(f"oracle check {'OK' if oracle_ok else 'MISMATCH'} ({time.time() - t1:.1f}s)")
            assert oracle_ok, (v_fused, want)
    summarize = getattr(w, "summary", lambda v: v)

    def barrier():
        if dist is not None:
            dist.barrier()
        ctx.synchronize()
        torch.cuda.synchronize(local)

    def timed(fn, steps, profile=False):
        for _ in range(args.warmup):
            fn()
        barrier()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        buf = (runq.C.c_char * 65536)()
        if profile:
            runq._L.rq_ctx_set_profiling(ctx.handle, 1)
            runq._L.rq_ctx_profile_report(ctx.handle, 1, buf, 65536)  # reset
        l0 = ctx.launches
        sampler = ClockSampler(local)
        with sampler:
            ev0.record(stream)
            for _ in range(steps):
                fn()
            if pending:  # the timed region ends when the last merge has landed
                with torch.cuda.stream(stream):
                    for _, h in pending:
                        h.wait()
            ev1.record(stream)
            ev1.synchronize()
        barrier()
        launches = ctx.launches - l0
        report = None
        if profile:
            runq._L.rq_ctx_profile_report(ctx.handle, 1, buf, 65536)
            runq._L.rq_ctx_set_profiling(ctx.handle, 0)
            report = json.loads(buf.value.decode())
        ms = ev0.elapsed_time(ev1) / steps
        if dist is not None:
            t = torch.tensor([ms], dtype=torch.float64, device=f"cuda:{local}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, launches, report, sampler.summary()

    # device-resident throughput (value) with live per-kernel event timing
    ms, launches, report, clocks = timed(lambda: step(dev, merge_async=True), args.steps, profile=True)
    pending.clear()
    value = world * rows / (ms / 1000.0)

    chain_ms = None
    if args.path == "fused":
        chain_ms, _, _, _ = timed(lambda: step(dev, "chain"), max(3, args.steps // 2))

    # e2e: upload compressed columns from pinned host memory + query + readback
    e2e = None
    if getattr(w, "chunked", False):
        e2e = {"value": None, "unit": UNIT, "h2d_bytes_per_step": None, "d2h_bytes_per_step": None,
               "note": "not measured: the chunked table is never whole in host memory"}
    elif not args.no_e2e:
        # only the columns the query reads cross PCIe
        used = getattr(w, "columns", None) or list(host)
        pinned = {k: pin_column(host[k]) for k in used}
        h2d = sum(col_bytes(v) for v in pinned.values())

        def e2e_step():
            d = {k: runq.upload(v, ctx) for k, v in pinned.items()}
            return step(d)

        e2e_ms, _, _, _ = timed(e2e_step, args.steps)
        e2e = {"value": world * rows / (e2e_ms / 1000.0), "unit": UNIT, "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": result_bytes(v_fused)}

    # roofline of the dominant tagged region (live CUDA-event timing)
    hbm, peak_kind = peaks()
    roof = None
    if report and w.tag in report:
        st = report[w.tag]
        avg_ms = st["ms"] / st["count"]
        ab = w.alg_bytes(host)
        achieved = ab / (avg_ms / 1000.0) / 1e9
        roof = {"bound": "hbm", "kernel": w.tag, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": ncu_traffic(w.name, w.tag), "alg_bytes_per_launch": ab,
                "avg_launch_ms": avg_ms, "launches": st["count"], "peak_source": peak_kind,
                "share_of_step": st["ms"] / (ms * args.steps)}
        if w.tag == "xg_rows":  # also the whole query (segment table + masks + row kernel) against its bytes
            w.tag = None
            qb = w.alg_bytes(host)
            w.tag = "xg_rows"
            roof["query_alg_bytes"] = qb
            roof["query_achieved_gbs"] = qb / (ms / 1000.0) / 1e9
            roof["query_traffic"] = ncu_traffic(w.name, "query")
    elif w.tag is None:  # operator-chain workloads: whole step against the query's bytes
        ab = w.alg_bytes(host)
        achieved = ab / (ms / 1000.0) / 1e9
        roof = {"bound": "hbm", "kernel": "query (operator chain)", "achieved": achieved, "peak": hbm,
                "unit": "GB/s", "frac": achieved / hbm, "traffic": ncu_traffic(w.name, "query"), "alg_bytes_per_launch": ab,
                "avg_launch_ms": ms, "launches": args.steps, "peak_source": peak_kind, "share_of_step": 1.0}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import refpy
        ref = refpy.Ref()
        sample_rows = min(rows, {"c3": 5_000_000, "q6": 60_000_000, "q1": 2_000_000,
                                 "c5": 20_000_000}.get(w.name, 200_000_000))
        from oracle.refpy import shard_column
        full = getattr(w, "cpu_sample", lambda h, r: None)(host, sample_rows)
        if full is not None:  # chunked table: a fresh table of the sample size, same generator
            sample = shard_map(full, 1)
        else:
            sample = shard_map({k: shard_column(v, 0, sample_rows) for k, v in host.items()}, 1)
        secs = []
        for _ in range(3):
            _, s = w.ref_run(ref, sample, 1)
            secs.append(s)
        sec = statistics.median(secs)
        cpu = {"value": sample_rows / sec, "unit": UNIT, "cores": 1, "kind": "reference",
               "sample": f"first {sample_rows} rows of the same table, reference operator chain "
                         f"(oracle/_ref) single-threaded, median of 3 ({sec:.2f}s)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": w.dtype, "data": "synthetic",
            "config": config_dict(args, w, rows), "e2e": e2e,
            "gpu_launches": launches, "roofline": roof, "cpu_baseline": cpu, "clocks": clocks,
            "chain_ms_per_step": chain_ms, "result": summarize(v_fused), "oracle_match": oracle_ok,
            "kernel_times_ms": report,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
