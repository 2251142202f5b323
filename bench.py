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

Multi-GPU (torchrun): one process per GPU. The N-GPU table is ONE table of
N × rows rows; each rank owns a row-range shard of it (cuts snapped to the run
boundaries of the column with the most runs; run-encoded columns cut with
rq_shard_host_column, plain columns generated for the rank's rows only), so
per-GPU work is fixed as N grows (weak scaling). Every step runs the
library's sharded entry point: the single-GPU kernels on the shard, then ONE
collective inside the library (NCCL all-reduce of the partial aggregates, or
an all-gather of the (key, partial) group tables + device regroup; AVG from
the merged SUM / COUNT). torch.distributed (gloo) only bootstraps the NCCL
unique id, barriers, and takes the max of the per-rank times. The gate
checks the merged result on rank 0 against the oracle of the whole table
(the merge of every rank's oracle over its own rows).

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
        clk = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        self.samples.append((time.perf_counter(), clk, r))

    def _run(self):
        # every 10 ms: NVML queries take driver locks that delay the launches
        # and syncs of host-paced steps (Q6 / C5: 27 launches per 0.4 ms step)
        while not self._stop.wait(0.01):
            self._sample()

    # The thread is started before the warm-up steps (its creation and first
    # NVML calls stay out of short timed regions); the summary keeps the
    # samples from 10 ms before the region to 10 ms after it.
    def __enter__(self):
        if self.ok:
            self._sample()
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def mark(self, start: bool):
        setattr(self, "t0" if start else "t1", time.perf_counter())

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()
            self._sample()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml-unavailable"]}
        t0, t1 = getattr(self, "t0", -1e30), getattr(self, "t1", 1e30)
        win = [x for x in self.samples if t0 - 0.01 <= x[0] <= t1 + 0.01] or self.samples
        reasons = sorted({name for _, _, r in win for bit, name in self.REASONS.items() if r & bit})
        return {"sm_mhz": float(statistics.median(c for _, c, _ in win)), "sm_max_mhz": float(self.max),
                "reasons": reasons, "samples": len(win)}


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


def stats_bytes(col):
    """The reference's own byte accounting, stats() (column.cpp:244-279):
    RLE R·(w+16) (positions s and e per run), Index P·(w+8), Plain storage
    bytes, composites summed — reported next to ALG_BYTES."""
    from paper_2506_10092_b200 import host as H
    if isinstance(col, H.RleColumn):
        return col.v.shape[0] * (col.v.itemsize + 16)
    if isinstance(col, H.IndexColumn):
        return col.p.shape[0] * (col.v.itemsize + 8)
    if isinstance(col, H.RlePlusIndexColumn):
        return stats_bytes(col.runs) + stats_bytes(col.points)
    if isinstance(col, H.PlainPlusIndexColumn):
        return stats_bytes(col.base) + stats_bytes(col.outliers)
    return col.values.nbytes


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


def f64_same(a, b):
    return abs(a - b) <= 1e-9 * max(1.0, abs(a), abs(b))


def scalar_partial(v):
    from oracle import streaming as S
    return S.Partial([], [np.array([v], np.int64)])


class Workload:
    """One BASELINE configuration. gen() returns this rank's shard of the
    table (the whole table when part is None); query() runs it through the
    library (sharded entry point when comm is given); oracle_partial() is the
    checker over the shard's rows, oracle_finish() of the merged partials is
    the whole table's expected result."""
    tag = None
    dtype = "int64"
    same = staticmethod(lambda a, b: a == b)
    summary = staticmethod(lambda v: v)
    chunked = False
    ref_rows = None

    def __init__(self, args):
        self.args = args

    def upload(self, rq, ctx, host, check):
        return {k: rq.upload(v, ctx) for k, v in host.items()}

    def oracle_finish(self, merged):
        return int(merged.parts[0][0])

    def stats_bytes(self, h):
        return sum(stats_bytes(c) for c in h.values())

    def cpu_sample(self, rows):
        return self.gen(rows, 42)

    def prepared(self, make, rq, d, comm):
        """The query's arguments marshalled once per table (agg.prepare_exprs,
        the call a repeated query makes); a new table (the e2e path uploads
        one per step) prepares again. Holds `d`, so its id cannot be reused."""
        if getattr(self, "_plan_for", None) is not d or getattr(self, "_plan_comm", None) is not comm:
            self._plan, self._plan_for, self._plan_comm = make(rq, d, comm), d, comm
        return self._plan


class C2(Workload):
    name = "c2"
    tag = "filtered_points_reduce"
    k = 20

    def describe(self):
        cdesc = "RLE L=256" if self.args.variant == "rle" else "plain-centered i8 L=4"
        return (f"C2: filtered SUM(A*B) WHERE C<{self.k}; A RLE i64 L=64, B Index i64 1%, "
                f"C dict codes (card 64) {cdesc}")

    def gen(self, rows, seed, part=None, slicer=None):
        from paper_2506_10092_b200 import datagen as G
        from paper_2506_10092_b200 import sharding
        a, b, c = G.c2_tables(rows, seed=seed, c_variant=self.args.variant)
        t = {"a": a, "b": b, "c": c}
        return t if part is None else sharding.shard_table(t, part[0], part[1], snap="a")

    def alg_bytes(self, h):
        from paper_2506_10092_b200 import host as H
        # C-rle R·16, C-narrow the whole predicate column n·1 B
        # (1.41 GB at 1B rows) — the kernel reads C only at B's points, so its
        # DRAM traffic (roofline.traffic) stays below that
        return alg_bytes(h["a"]) + alg_bytes(h["b"]) + alg_bytes(h["c"])

    def query(self, rq, d, path, comm=None):
        if path == "fused":  # arguments marshalled once per table (agg.prepare_filtered_binop)
            return self.prepared(lambda rq_, t, cm: rq_.agg.prepare_filtered_binop(t["c"], self.k, "<", t["a"], t["b"],
                                                                                  "*", "sum", comm=cm), rq, d, comm)()
        m = rq.compute.compare_scalar(d["c"], self.k, "<")
        return rq.agg.aggregate_all(rq.compute.arith(rq.compute.filter(d["a"], m), rq.compute.filter(d["b"], m), "*"),
                                    "sum", comm=comm)

    def oracle_partial(self, h):
        from oracle import refpy
        return scalar_partial(refpy.Orq().filtered_sum(h["c"], self.k, "<", h["a"], h["b"], "*"))

    def ref_run(self, ref, shards, threads):
        return ref.chain_filtered_sum(shards["c"], shards["a"], shards["b"], threads, self.k, "<", "*")


class C1(Workload):
    name = "c1"
    tag = "pair_reduce"

    def describe(self):
        la, lb = getattr(self.args, "c1_runs", (64, 96))
        return f"C1: SUM(A+B) over two misaligned RLE i64 columns, L={la}/{lb}"

    def gen(self, rows, seed, part=None, slicer=None):
        from paper_2506_10092_b200 import datagen as G
        from paper_2506_10092_b200 import sharding
        la, lb = getattr(self.args, "c1_runs", (64, 96))
        a, b = G.c1_tables(rows, la, lb, seed)
        t = {"a": a, "b": b}
        return t if part is None else sharding.shard_table(t, part[0], part[1], snap="a")

    def alg_bytes(self, h):
        return alg_bytes(h["a"]) + alg_bytes(h["b"])

    def query(self, rq, d, path, comm=None):
        if path == "fused":  # arguments marshalled once per table (agg.prepare_binop)
            return self.prepared(lambda rq_, t, cm: rq_.agg.prepare_binop(t["a"], t["b"], "+", "sum", comm=cm),
                                 rq, d, comm)()
        return rq.agg.aggregate_all(rq.compute.arith(d["a"], d["b"], "+"), "sum", comm=comm)

    def oracle_partial(self, h):
        from oracle import refpy
        return scalar_partial(refpy.Orq().sum_rle_binop(h["a"], h["b"], "+"))

    def ref_run(self, ref, shards, threads):
        return ref.chain_sum_binop(shards["a"], shards["b"], threads, "+")


class C3(Workload):
    name = "c3"
    tag = "group_fused"
    dtype = "int64/f64"
    host_rows_max = 2_000_000_000  # above this Z / W stream into HBM chunk by chunk (never whole on the host)
    same = staticmethod(tables_same)
    summary = staticmethod(table_summary)
    ref_rows = 20_000_000

    def __init__(self, args):
        super().__init__(args)
        self.fold = None

    def describe(self):
        return ("C3: GROUP BY K (codes 0..99, RLE L=4096) -> SUM(X RLE L=128), COUNT(*), AVG(Z plain-centered i16), "
                "SUM(Y RLE+Index 90% runs L=256 / 10% points), SUM(W plain f64)")

    def gen(self, rows, seed, part=None, slicer=None):
        from paper_2506_10092_b200 import datagen as G
        from paper_2506_10092_b200 import host as H
        k, x, y, lo, hi = G.c3_run_columns(rows, seed, part, slicer)
        self.total, self.seed, self.lo, self.hi = rows, seed, lo, hi
        self.chunked = hi - lo > self.host_rows_max
        t = {"k": k, "x": x, "y": y}
        if not self.chunked:
            z, w = G.c3_plain_rows(rows, seed, lo, hi)
            t["z"], t["w"] = H.PlainColumn(z, H.I64, 0), H.PlainColumn(w)
        return t

    def upload(self, rq, ctx, host, check):
        """Chunked shards: Z / W generated chunk by chunk, written into HBM
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
        n = self.hi - self.lo
        za, wa = rq.alloc_array(H.I16, n, ctx), rq.alloc_array(H.F64, n, ctx)
        t0 = time.time()
        r = self.lo
        while r < self.hi:
            r1 = min(self.hi, (r // G.GEN_CHUNK + 1) * G.GEN_CHUNK)
            z, w = G.c3_plain_rows(self.total, self.seed, r, r1)
            keep = (za.write(r - self.lo, z), wa.write(r - self.lo, w))
            if self.fold is not None:
                self.fold.add_plain_chunk(r - self.lo, H.PlainColumn(z, H.I64, 0), w)
            ctx.synchronize()
            del keep
            r = r1
        log(f"streamed Z/W ({n} rows) into HBM in {time.time() - t0:.1f}s")
        dev["z"], dev["w"] = rq.make_plain(za, H.I64, 0), rq.make_plain(wa)
        return dev

    def alg_bytes(self, h):
        b = sum(alg_bytes(h[n]) for n in ("k", "x", "y"))
        return b + (self.hi - self.lo) * (2 + 8)  # Z i16 + W f64 per row

    def stats_bytes(self, h):
        return sum(stats_bytes(h[n]) for n in ("k", "x", "y")) + (self.hi - self.lo) * (2 + 8)

    def query(self, rq, d, path, comm=None):
        from paper_2506_10092_b200 import datagen as G
        ks, vs, ng = rq.agg.group_aggregate([d["k"]], [d["x"], d["k"], d["z"], d["y"], d["w"]], G.C3_FNS,
                                            normalize=True, comm=comm)
        h = rq.download_all(list(ks) + list(vs))
        return h[:1], h[1:]

    def oracle_partial(self, h):
        """The streaming oracle (oracle/streaming.py, pinned against the
        reference library up to 100M rows) over this shard's rows."""
        from oracle import streaming as S
        if self.fold is not None:
            return self.fold.partial()
        return S.c3_partial(h)

    def oracle_finish(self, merged):
        from oracle import streaming as S
        return S.c3_finish(merged)

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


class Q6(Workload):
    """C4: TPC-H-style Q6 over synthetic lineitem (SF = rows / 6M) sorted by
    (quantity, discount, shipdate)."""
    name = "q6"
    dtype = "f64"
    ref_rows = 60_000_000  # reference arm sample (SF10)
    same = staticmethod(f64_same)

    def __init__(self, args):
        super().__init__(args)
        # fused path: the K12 row kernel (the query's dominant kernel); chain: whole query
        self.tag = "xg_rows" if args.path == "fused" else None

    def describe(self):
        return (f"C4 Q6: SUM(price*disc) WHERE shipdate in [1994-01-01,1995-01-01) AND disc BETWEEN 5 AND 7 AND "
                f"qty < 24; lineitem SF{self.args.rows / 6e6:g} per GPU sorted (qty, disc, shipdate), RLE keys + "
                f"f64 price")

    def gen(self, rows, seed, part=None, slicer=None):
        from paper_2506_10092_b200 import queries as Q
        return Q.lineitem_q6(rows, seed, part, slicer)

    def alg_bytes(self, h):
        sd, d, q = h["l_shipdate"], h["l_discount"], h["l_quantity"]
        # price is read only at the selected rows: estimate them from the runs
        sel = self._selected(h)
        if self.tag == "xg_rows":  # the row kernel reads price at the selected rows
            return sel * 8
        return alg_bytes(sd) + alg_bytes(d) + alg_bytes(q) + sel * 8

    def _selected(self, h):
        from paper_2506_10092_b200 import queries as Q
        sd, d, q = h["l_shipdate"], h["l_discount"], h["l_quantity"]
        sds = sd.s if sd.s is not None else np.concatenate([[0], sd.e[:-1] + 1])
        qi = np.searchsorted(q.e, sds)
        di = np.searchsorted(d.e, sds)
        ok = (q.v[qi] < 24) & (d.v[di] >= 5) & (d.v[di] <= 7) & (sd.v >= Q.Q6_LO) & (sd.v < Q.Q6_HI)
        return int((sd.e - sds + 1)[ok].sum())

    def query(self, rq, d, path, comm=None):
        from paper_2506_10092_b200 import queries as Q
        if path == "fused":
            v, fused = self.prepared(Q.q6_prepared, rq, d, comm)()
            assert fused, "q6: fused path not taken"
            return v
        return Q.q6(rq, d)

    def oracle_partial(self, h):
        from oracle import streaming as S
        from paper_2506_10092_b200 import queries as Q
        return S.q6_partial(h, Q.Q6_WHERE)

    def oracle_finish(self, merged):
        from oracle import streaming as S
        return S.q6_finish(merged)

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
    same = staticmethod(tables_same)
    summary = staticmethod(table_summary)

    def describe(self):
        return (f"C4 Q1: GROUP BY returnflag, linestatus: 4 SUMs, 3 AVGs, COUNT WHERE shipdate <= 1998-09-02; "
                f"lineitem SF{self.args.rows / 6e6:g} per GPU sorted (rf, ls, shipdate, qty); disc/tax i8 plain, "
                f"price f64")

    def gen(self, rows, seed, part=None, slicer=None):
        from paper_2506_10092_b200 import queries as Q
        return Q.lineitem_q1(rows, seed + 1, part, slicer)

    def alg_bytes(self, h):
        if self.tag == "xg_rows":  # the row kernel streams price / disc / tax over the rows passing the filter
            from paper_2506_10092_b200 import queries as Q
            sd = h["l_shipdate"]
            sds = sd.s if sd.s is not None else np.concatenate([[0], sd.e[:-1] + 1])
            sel = int((sd.e - sds + 1)[sd.v <= Q.Q1_CUTOFF].sum())
            return sel * (8 + 1 + 1)
        return sum(alg_bytes(c, gapless=True) for c in h.values())

    def query(self, rq, d, path, comm=None):
        from paper_2506_10092_b200 import queries as Q
        if path == "fused":
            (ks, vs, ng), fused = self.prepared(Q.q1_prepared, rq, d, comm)()
            assert fused, "q1: fused path not taken"
        else:
            ks, vs, ng = Q.q1(rq, d)
        h = rq.download_all(list(ks) + list(vs))
        return h[:2], h[2:]

    def oracle_partial(self, h):
        from oracle import streaming as S
        from paper_2506_10092_b200 import queries as Q
        return S.q1_partial(h, Q.Q1_CUTOFF)

    def oracle_finish(self, merged):
        from oracle import streaming as S
        return S.q1_finish(merged)

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
    750M rows per GPU: 6B rows over 8 GPUs (the table is too large
    uncompressed for one GPU)."""
    name = "c5"
    dtype = "int64"
    same = staticmethod(tables_same)
    summary = staticmethod(table_summary)
    ref_rows = 20_000_000
    columns = ["r2", "r3", "r4", "pi0", "p1"]

    def describe(self):
        return ("C5: production-shaped 15 cols (7 RLE i32 codes, 4 Plain+Index i16+1% i64, 4 narrow plain); "
                "WHERE r2 IN (3,17,42) AND r3 < 50 GROUP BY r4 -> SUM(pi0), SUM(p1), COUNT(*); the columns the "
                "query reads are generated")

    def gen(self, rows, seed, part=None, slicer=None):
        from paper_2506_10092_b200 import queries as Q
        return Q.production_table(rows, seed - 37, part, slicer, columns=self.columns)

    def alg_bytes(self, h):
        # predicate / key runs + the two measures read only at the selected rows
        sel = getattr(self, "_sel", 0)
        runs = sum(alg_bytes(h[k]) for k in ("r2", "r3", "r4"))
        pi0 = h["pi0"]
        if self.tag == "xg_rows":  # the row kernel reads the two i16 measures at the selected rows
            return sel * (2 + 2)
        out_frac = len(pi0.outliers.p) / max(1, pi0.base.values.shape[0])
        return runs + sel * (2 + 2) + int(sel * out_frac) * 16

    def query(self, rq, d, path, comm=None):
        from paper_2506_10092_b200 import queries as Q
        if path == "fused":
            (ks, vs, ng), fused = self.prepared(Q.c5_prepared, rq, d, comm)()
            assert fused, "c5: fused path not taken"
        else:
            ks, vs, ng = Q.c5_query(rq, d)
        h = rq.download_all(list(ks) + list(vs))
        self._sel = int(h[3].sum())  # selected rows (COUNT column): the measures are read only there
        return h[:1], h[1:]

    def oracle_partial(self, h):
        from oracle import streaming as S
        from paper_2506_10092_b200 import queries as Q
        return S.c5_partial(h, Q.C5_IN, Q.C5_LT)

    def oracle_finish(self, merged):
        from oracle import streaming as S
        return S.c5_finish(merged)

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


def config_dict(args, w, rows, world=1):
    return {"workload": w.describe(), "rows_per_gpu": rows, "total_rows": rows * world, "query_path": args.path,
            "sharding": ("one table of rows_per_gpu x N rows, row-range shards (cuts snapped to runs), one "
                         "in-library collective per step" if world > 1 else "single GPU"),
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
    rows = min(args.rows, w.ref_rows or args.rows)
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
                    help="logical rows per GPU (default 1B; SF100 = 600M for q6/q1; 750M for c5)")
    ap.add_argument("--variant", default="rle", choices=["rle", "narrow"])
    ap.add_argument("--c1-runs", default="64,96", help="C1 mean run lengths of A,B (SURVEY §8d sweep: 16,24 / 64,96 / 1000,1500)")
    ap.add_argument("--path", default="fused", choices=["fused", "chain"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--comm", default="nccl", choices=["nccl", "host"],
                    help="N>1 transport: the library's NCCL communicator (one rank per GPU), or its host "
                         "transport over gloo (several ranks may share a GPU: tests of the N>1 logic)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    args.c1_runs = tuple(int(x) for x in args.c1_runs.split(","))
    if args.rows is None:
        args.rows = {"q6": 600_000_000, "q1": 600_000_000, "c5": 750_000_000}.get(args.workload, 1_000_000_000)
    w = WORKLOADS[args.workload](args)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        # plumbing only (unique-id broadcast, barriers, max-over-ranks time,
        # oracle partials); the data-path collective is the library's NCCL
        import torch.distributed as dist
        dist.init_process_group("gloo")

    if args.impl == "reference":
        run_reference(args, w, rank, world)
        if dist is not None:
            dist.destroy_process_group()
        return

    import torch
    from paper_2506_10092_b200 import runq

    rows = args.rows
    total = rows * world
    t0 = time.time()
    part = (rank, world) if world > 1 else None
    host = w.gen(total, 42, part, runq.shard_host_column)
    log(f"[rank {rank}] generated {w.name}: shard of {total} rows in {time.time() - t0:.1f}s")

    if args.comm == "host":  # ranks may share a device
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    ctx = runq.Context(local)
    stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", local))
    comm = None
    if world > 1 and args.comm == "nccl":
        uid = [runq.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = runq.Comm.nccl(ctx, uid[0], world, rank)
    elif world > 1:
        def allgather(b):
            out = [None] * world
            dist.all_gather_object(out, b)
            return out
        comm = runq.Comm.host(ctx, world, rank, allgather)
    check = True  # every rank folds its shard's oracle; rank 0 merges them
    dev = w.upload(runq, ctx, host, check)

    # correctness gate: fused == device chain (N=1) and merged result == the
    # oracle of the whole table (rank 0). The oracle is the C restatement
    # (C1 / C2) or the streaming group-by oracle (C3 / Q1 / Q6 / C5,
    # oracle/streaming.py), pinned against the reference library up to 100M
    # rows; for N>1 it is the merge of every rank's oracle over its own rows.
    same = w.same
    v_fused = w.query(runq, dev, args.path, comm)
    if args.path == "fused" and world == 1:  # fused kernels == the device operator chain
        v_chain = w.query(runq, dev, "chain")
        assert same(v_fused, v_chain), (v_fused, v_chain)
    t1 = time.time()
    mine = w.oracle_partial(host)
    parts = [mine]
    if dist is not None:
        parts = [None] * world
        dist.all_gather_object(parts, mine)
    from oracle import streaming as S
    want = w.oracle_finish(S.merge(parts))
    oracle_ok = bool(same(v_fused, want))
    if rank == 0:
        log(f"oracle check {'OK' if oracle_ok else 'MISMATCH'} ({time.time() - t1:.1f}s)")
    assert oracle_ok, (v_fused, want)

    def barrier():
        ctx.synchronize()
        torch.cuda.synchronize(local)
        if dist is not None:
            dist.barrier()

    def timed(fn, steps, profile=False):
        sampler = ClockSampler(local)
        buf = (runq.C.c_char * 65536)()
        if profile:
            # only the dominant kernel's region is timed live (two events per
            # step): per-scope events would add their own cost to small queries.
            # On from the warm-up on: the warm-up calls then build the same
            # plan (and CUDA graph) the timed calls run.
            runq._L.rq_ctx_profile_only(ctx.handle, profile.encode())
            runq._L.rq_ctx_set_profiling(ctx.handle, 1)
        with sampler:
            for _ in range(args.warmup):
                fn()
            barrier()
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            if profile:
                runq._L.rq_ctx_profile_report(ctx.handle, 1, buf, 65536)  # reset: timed steps only
            l0 = ctx.launches
            sampler.mark(True)
            ev0.record(stream)
            for _ in range(steps):
                fn()
            ev1.record(stream)
            ev1.synchronize()
            sampler.mark(False)
        barrier()
        launches = ctx.launches - l0
        report = None
        if profile:
            runq._L.rq_ctx_profile_report(ctx.handle, 1, buf, 65536)
            runq._L.rq_ctx_set_profiling(ctx.handle, 0)
            report = json.loads(buf.value.decode())
        ms = ev0.elapsed_time(ev1) / steps
        if dist is not None:  # max over ranks
            t = torch.tensor([ms], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, launches, report, sampler.summary()

    # device-resident throughput (value) with live per-kernel event timing
    ms, launches, report, clocks = timed(lambda: w.query(runq, dev, args.path, comm), args.steps,
                                         profile=w.tag or False)
    value = total / (ms / 1000.0)

    chain_ms = None
    if args.path == "fused" and world == 1:
        chain_ms, _, _, _ = timed(lambda: w.query(runq, dev, "chain"), max(3, args.steps // 2))

    # e2e: upload the shard's compressed columns from pinned host memory +
    # query + readback of the merged result
    e2e = None
    if w.chunked:
        e2e = {"value": None, "unit": UNIT, "h2d_bytes_per_step": None, "d2h_bytes_per_step": None,
               "note": "not measured: the chunked table is never whole in host memory"}
    elif not args.no_e2e:
        pinned = {k: pin_column(v) for k, v in host.items()}
        h2d = sum(col_bytes(v) for v in pinned.values())

        def e2e_step():
            d = {k: runq.upload(v, ctx) for k, v in pinned.items()}
            return w.query(runq, d, args.path, comm)

        e2e_ms, _, _, _ = timed(e2e_step, args.steps)
        e2e = {"value": total / (e2e_ms / 1000.0), "unit": UNIT, "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": result_bytes(v_fused)}

    # roofline of the dominant tagged region (live CUDA-event timing, this rank)
    hbm, peak_kind = peaks()
    roof = None
    if report and w.tag in report:
        st = report[w.tag]
        avg_ms = st["ms"] / st["count"]
        ab = w.alg_bytes(host)
        achieved = ab / (avg_ms / 1000.0) / 1e9
        roof = {"bound": "hbm", "kernel": w.tag, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": ncu_traffic(w.name + ("_narrow" if args.variant == "narrow" else ""), w.tag),
                "alg_bytes_per_launch": ab,
                "stats_bytes": w.stats_bytes(host), "avg_launch_ms": avg_ms, "launches": st["count"],
                "peak_source": peak_kind, "share_of_step": st["ms"] / (ms * args.steps)}
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
                "unit": "GB/s", "frac": achieved / hbm, "traffic": ncu_traffic(w.name, "query"),
                "alg_bytes_per_launch": ab, "stats_bytes": w.stats_bytes(host), "avg_launch_ms": ms,
                "launches": args.steps, "peak_source": peak_kind, "share_of_step": 1.0}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import refpy
        ref = refpy.Ref()
        sample_rows = min(rows, {"c3": 5_000_000, "q6": 60_000_000, "q1": 2_000_000,
                                 "c5": 20_000_000}.get(w.name, 200_000_000))
        sample = shard_map(w.cpu_sample(sample_rows), 1)
        secs = []
        for _ in range(3):
            _, s = w.ref_run(ref, sample, 1)
            secs.append(s)
        sec = statistics.median(secs)
        cpu = {"value": sample_rows / sec, "unit": UNIT, "cores": 1, "kind": "reference",
               "sample": f"a {sample_rows}-row table of the same generator, reference operator chain "
                         f"(oracle/_ref) single-threaded, median of 3 ({sec:.2f}s)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": w.dtype, "data": "synthetic",
            "config": config_dict(args, w, rows, world), "e2e": e2e,
            "gpu_launches": launches, "roofline": roof, "cpu_baseline": cpu, "clocks": clocks,
            "chain_ms_per_step": chain_ms, "result": w.summary(v_fused), "oracle_match": oracle_ok,
            "collective": (None if world == 1 else
                           "library NCCL (rq_comm_init_nccl): grouped all-reduce of partials / all-gather of "
                           "group tables + device regroup, inside the timed step" if args.comm == "nccl" else
                           "library host transport over gloo (test mode)"),
            "kernel_times_ms": report,
        }
        print(json.dumps(line), flush=True)
    del comm
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
