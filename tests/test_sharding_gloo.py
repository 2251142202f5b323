"""CPU, world size 2 over gloo: the multi-GPU path's host logic — row-range
shard planning, per-rank execution on standalone shards, and the
single-collective merge — reproduces the unsharded result. Per-rank compute
uses the reference library (the checker) so this runs without a GPU; on the
B200 box the same shards run through the device path (bench.py)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2506_10092_b200 import datagen as G
from paper_2506_10092_b200 import sharding as S


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import refpy
        ref = refpy.Ref()
        # C2 chain on this rank's shard, merged with one all_reduce
        a, b, c = G.c2_tables(400_000, seed=11)
        sh = S.shard_table({"a": a, "b": b, "c": c}, rank, world, snap="a")
        m = ref.compare_scalar(sh["c"], 20, "<")
        part = ref.aggregate_all(ref.arith(ref.filter(sh["a"], m), ref.filter(sh["b"], m), "*"), "sum")
        total = S.allreduce_scalar_i64(part)
        # C1: SUM(A+B) and COUNT via partials
        a1, b1 = G.c1_tables(300_000, 16, 24, seed=5)
        sh1 = S.shard_table({"a": a1, "b": b1}, rank, world)
        s1 = S.allreduce_scalar_i64(ref.aggregate_all(ref.arith(sh1["a"], sh1["b"], "+"), "sum"))
        # group-by: per-rank (keys, SUM, COUNT) tables, all_gather, merge
        k, x, y, z, w = G.c3_tables(200_000, seed=3)
        sh3 = S.shard_table({"k": k, "x": x, "z": z}, rank, world)
        ks, vs, _ = ref.group_aggregate([sh3["k"]], [sh3["x"], sh3["k"], sh3["z"]], ["sum", "count", "sum"])
        gathered = [None] * world
        dist.all_gather_object(gathered, (ks[0], vs[0], vs[1], vs[2]))
        uk, sx, cnt = S.merge_group_tables([g[0] for g in gathered], [g[1] for g in gathered],
                                           [g[2] for g in gathered])
        _, sz, _ = S.merge_group_tables([g[0] for g in gathered], [g[3] for g in gathered],
                                        [g[2] for g in gathered])
        if rank == 0:
            q.put((total, s1, uk, sx, cnt, sz / cnt))
    finally:
        dist.destroy_process_group()


def test_two_rank_shard_and_merge(ref):
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    total, s1, uk, sx, cnt, avg_z = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a, b, c = G.c2_tables(400_000, seed=11)
    m = ref.compare_scalar(c, 20, "<")
    assert total == ref.aggregate_all(ref.arith(ref.filter(a, m), ref.filter(b, m), "*"), "sum")
    a1, b1 = G.c1_tables(300_000, 16, 24, seed=5)
    assert s1 == ref.aggregate_all(ref.arith(a1, b1, "+"), "sum")
    k, x, y, z, w = G.c3_tables(200_000, seed=3)
    wk, wv, _ = ref.group_aggregate([k], [x, k, z], ["sum", "count", "avg"])
    assert np.array_equal(uk, wk[0])
    assert np.array_equal(sx, wv[0])
    assert np.array_equal(cnt, wv[1])
    assert np.allclose(avg_z, wv[2], rtol=1e-12)


def test_plan_cuts_snap_and_merge_rules():
    a = G.gapless_rle(10_000, 64, 1)
    cuts = S.plan_cuts(10_000, 4, a)
    assert cuts[0] == 0 and cuts[-1] == 10_000 and len(cuts) == 5
    ends = set((a.e + 1).tolist())
    assert all(c in ends for c in cuts[1:-1])
    # int64 SUM wraps exactly like the reference accumulator
    big = np.iinfo(np.int64).max
    assert S.merge_scalar([big, 1], "sum") == np.iinfo(np.int64).min
    assert S.merge_scalar([2.0, 4.0], "avg", counts=[1, 2]) == 2.0
