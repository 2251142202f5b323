#!/usr/bin/env python
"""Benchmark of the compressed-execution query path (BASELINE.json metric:
logical rows/s per query and % of HBM roofline on compressed bytes).

Default workload = BASELINE config[1] (C2): filtered SUM(A*B) WHERE C < k
over 1B logical rows per GPU — A RLE int64 (L=64, 15.6M runs), B Index int64
(1% density, 10M points), C dictionary codes (cardinality 64) RLE L=256.
A step is one execution of the query through the C ABI
(rq_filtered_aggregate_binop → the fused single-pass kernel) on
device-resident compressed columns; `e2e` repeats it through the same call
with the compressed columns uploaded from pinned host memory every step and
the result read back. Inputs (0.47 GB/GPU) exceed L2 (126 MB), so no flush is
needed between steps.

Multi-GPU (torchrun): one process per GPU, each rank owns a 1B-row range
shard of an N-billion-row table (weak scaling); the per-rank partial SUM is
merged with one NCCL all_reduce per step.

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
        while not self._stop.is_set():
            self._sample()
            time.sleep(0.002)

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
        return H.RleColumn(pinned_copy(col.v), pinned_copy(col.s), pinned_copy(col.e), col.total_size)
    if isinstance(col, H.IndexColumn):
        return H.IndexColumn(pinned_copy(col.v), pinned_copy(col.p), col.total_size)
    if isinstance(col, H.PlainColumn):
        return H.PlainColumn(pinned_copy(col.values), col.logical, col.center)
    raise TypeError(type(col))


def col_bytes(col):
    from paper_2506_10092_b200 import host as H
    if isinstance(col, H.RleColumn):
        return col.v.nbytes + col.s.nbytes + col.e.nbytes
    if isinstance(col, H.IndexColumn):
        return col.v.nbytes + col.p.nbytes
    return col.values.nbytes


def alg_bytes_c2(a, b, c):
    """ALG_BYTES: gapless RLE R·(w_v+8) (v + e), Index
    P·(w_v+8), a plain column read only at B's points P·w_storage."""
    from paper_2506_10092_b200 import host as H
    ab = a.v.shape[0] * (a.v.itemsize + 8)
    bb = b.p.shape[0] * (b.v.itemsize + 8)
    if isinstance(c, H.RleColumn):
        cb = c.v.shape[0] * (c.v.itemsize + 8)
    else:
        cb = b.p.shape[0] * c.values.itemsize
    return ab + bb + cb


def ncu_traffic(tag):
    """dram bytes per launch of the dominant kernel from the committed ncu
    capture summary (profiles/ncu_traffic.json), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(tag, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------


def shard_list(col, nshards):
    from paper_2506_10092_b200.runq import shard_host_column
    n = col.total_size
    cuts = [n * i // nshards for i in range(nshards + 1)]
    return [shard_host_column(col, lo, hi) for lo, hi in zip(cuts[:-1], cuts[1:])]


def run_reference(args, rank, world):
    if rank != 0:
        return
    from oracle import refpy
    from paper_2506_10092_b200 import datagen as G
    ref = refpy.Ref()
    threads = os.cpu_count() or 1
    rows = args.rows
    a, b, c = G.c2_tables(rows, seed=42, c_variant=args.variant)
    nshards = threads
    cs, as_, bs = shard_list(c, nshards), shard_list(a, nshards), shard_list(b, nshards)
    for _ in range(args.warmup):
        ref.chain_filtered_sum(cs, as_, bs, threads, G.C2_K, "<", "*")
    times = []
    for _ in range(args.steps):
        val, sec = ref.chain_filtered_sum(cs, as_, bs, threads, G.C2_K, "<", "*")
        times.append(sec)
    ms = 1000.0 * statistics.median(times)
    value = rows / (ms / 1000.0)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic",
        "config": config_dict(args, rows),
        "result": val,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"full {rows:.0f}-row table as {nshards} row-range shards on {threads} threads "
                                   "(reference operator chain compare_scalar→filter×2→arith→aggregate_all per shard)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_dict(args, rows):
    cdesc = "RLE L=256" if args.variant == "rle" else "plain-centered i8 L=4"
    return {"workload": f"C2: filtered SUM(A*B) WHERE C<20; A RLE i64 L=64, B Index i64 1%, C dict codes "
                        f"(card 64) {cdesc}", "rows_per_gpu": rows, "query_path": args.path,
            "l2_policy": "inputs larger than L2 (126 MB) — no flush needed"}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--rows", type=int, default=1_000_000_000)
    ap.add_argument("--variant", default="rle", choices=["rle", "narrow"])
    ap.add_argument("--path", default="fused", choices=["fused", "chain"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl" if args.impl == "ours" else "gloo",
                                device_id=torch.device("cuda", local) if args.impl == "ours" else None)

    if args.impl == "reference":
        run_reference(args, rank, world)
        if dist is not None:
            dist.destroy_process_group()
        return

    import torch
    from paper_2506_10092_b200 import datagen as G
    from paper_2506_10092_b200 import runq

    rows = args.rows
    t0 = time.time()
    a, b, c = G.c2_tables(rows, seed=42 + rank, c_variant=args.variant)
    log(f"[rank {rank}] generated {rows} rows in {time.time() - t0:.1f}s: A runs={len(a.s)} "
        f"B points={len(b.p)} C={'runs=%d' % len(c.s) if hasattr(c, 's') else 'rows=%d' % c.total_size}")

    ctx = runq.Context(local)
    stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", local))
    da, db, dc = runq.upload(a, ctx), runq.upload(b, ctx), runq.upload(c, ctx)
    k = G.C2_K

    def query(xc, xa, xb):
        if args.path == "fused":
            return runq.agg.filtered_aggregate_binop(xc, k, "<", xa, xb, "*", "sum")
        m = runq.compute.compare_scalar(xc, k, "<")
        return runq.agg.aggregate_all(
            runq.compute.arith(runq.compute.filter(xa, m), runq.compute.filter(xb, m), "*"), "sum")

    red = torch.zeros(1, dtype=torch.int64, device=f"cuda:{local}")

    def step(xc, xa, xb):
        v = query(xc, xa, xb)
        if dist is not None:  # partial-aggregate merge over NCCL (int64 SUM wraps like the reference)
            red.fill_(v)
            dist.all_reduce(red)
            v = int(red.item())
        return v

    # correctness gate: fused == device chain == C oracle (rank 0, N=1)
    v_fused = runq.agg.filtered_aggregate_binop(dc, k, "<", da, db, "*", "sum")
    m = runq.compute.compare_scalar(dc, k, "<")
    v_chain = runq.agg.aggregate_all(runq.compute.arith(runq.compute.filter(da, m), runq.compute.filter(db, m), "*"), "sum")
    del m
    assert v_fused == v_chain, (v_fused, v_chain)
    oracle_ok = None
    if rank == 0 and world == 1:
        from oracle import refpy
        t1 = time.time()
        want = refpy.Orq().filtered_sum(c, k, "<", a, b, "*")
        oracle_ok = want == v_fused
        log(f"oracle check {'OK' if oracle_ok else 'MISMATCH'} ({time.time() - t1:.1f}s): {v_fused} vs {want}")
        assert oracle_ok

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
        if profile:
            runq._L.rq_ctx_set_profiling(ctx.handle, 1)
            buf = (runq.C.c_char * 65536)()
            runq._L.rq_ctx_profile_report(ctx.handle, 1, buf, 65536)  # reset
        l0 = ctx.launches
        sampler = ClockSampler(local)
        with sampler:
            ev0.record(stream)
            for _ in range(steps):
                fn()
            ev1.record(stream)
            ev1.synchronize()
        barrier()
        launches = ctx.launches - l0
        report = None
        if profile:
            buf = (runq.C.c_char * 65536)()
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
    ms, launches, report, clocks = timed(lambda: step(dc, da, db), args.steps, profile=True)
    value = world * rows / (ms / 1000.0)

    # chain path for reference (same inputs, same result)
    chain_ms = None
    if args.path == "fused":
        saved = args.path
        args.path = "chain"
        chain_ms, _, _, _ = timed(lambda: step(dc, da, db), max(3, args.steps // 2))
        args.path = saved

    # e2e: upload compressed columns from pinned host memory + query + readback
    pa, pb, pc = pin_column(a), pin_column(b), pin_column(c)
    h2d = col_bytes(pa) + col_bytes(pb) + col_bytes(pc)

    def e2e_step():
        xa, xb, xc = runq.upload(pa, ctx), runq.upload(pb, ctx), runq.upload(pc, ctx)
        return step(xc, xa, xb)

    e2e_ms, _, _, _ = timed(e2e_step, args.steps)
    e2e_value = world * rows / (e2e_ms / 1000.0)

    # roofline of the dominant kernel (live CUDA-event timing from the library)
    hbm, peak_kind = peaks()
    dom = max(report.items(), key=lambda kv: kv[1]["ms"]) if report else (None, None)
    roof = None
    if dom[0]:
        tag, st = dom
        avg_ms = st["ms"] / st["count"]
        ab = alg_bytes_c2(a, b, c) if tag == "filtered_points_reduce" else None
        achieved = ab / (avg_ms / 1000.0) / 1e9 if ab else None
        roof = {"bound": "hbm", "kernel": tag, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm if achieved else None, "traffic": ncu_traffic(tag),
                "alg_bytes_per_launch": ab, "avg_launch_ms": avg_ms, "launches": st["count"],
                "peak_source": peak_kind, "share_of_step": st["ms"] / (ms * args.steps)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import refpy
        ref = refpy.Ref()
        sample_rows = min(rows, 200_000_000)
        from paper_2506_10092_b200.runq import shard_host_column
        sa = shard_host_column(a, 0, sample_rows)
        sb = shard_host_column(b, 0, sample_rows)
        sc = shard_host_column(c, 0, sample_rows)
        secs = []
        for _ in range(3):
            _, s = ref.chain_filtered_sum([sc], [sa], [sb], 1, k, "<", "*")
            secs.append(s)
        sec = statistics.median(secs)
        cpu = {"value": sample_rows / sec, "unit": UNIT, "cores": 1, "kind": "reference",
               "sample": f"first {sample_rows} rows of the same table, reference operator chain "
                         f"(oracle/_ref) single-threaded, median of 3 ({sec:.2f}s)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": config_dict(args, rows),
            "e2e": {"value": e2e_value, "unit": UNIT, "ms_per_step": e2e_ms, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": 8},
            "gpu_launches": launches, "roofline": roof, "cpu_baseline": cpu, "clocks": clocks,
            "chain_ms_per_step": chain_ms, "result": v_fused, "oracle_match": oracle_ok,
            "kernel_times_ms": report,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
