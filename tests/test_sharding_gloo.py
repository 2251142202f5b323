"""CPU, world size 2 over gloo: the multi-GPU path's host logic — row-range
shard planning (plan_cuts, snapped to run boundaries), every rank generating
ONLY its shard of one table (datagen part=(rank, world), run columns cut by
the product's rq_shard_host_column — a pure host function of the C ABI),
per-rank execution on the standalone shard, and the merge of per-rank partial
results — reproduces the reference's UNSHARDED result. Per-rank compute here
is the reference library (the checker) and the merge is the oracle's, so this
runs without a GPU; the device path with the library's own merge runs two
ranks on cuda:0 in tests/test_gpu_sharded.py, and NCCL at N GPUs in bench.py."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2506_10092_b200 import datagen as G
from paper_2506_10092_b200 import queries as Q
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
        from oracle import streaming as O
        from paper_2506_10092_b200 import runq
        ref = refpy.Ref()
        slicer = runq.shard_host_column
        out = {}
        # C2 chain on this rank's shard: one int64 partial
        a, b, c = G.c2_tables(400_000, seed=11)
        sh = S.shard_table({"a": a, "b": b, "c": c}, rank, world, snap="a")
        m = ref.compare_scalar(sh["c"], 20, "<")
        out["c2"] = ref.aggregate_all(ref.arith(ref.filter(sh["a"], m), ref.filter(sh["b"], m), "*"), "sum")
        # C3: this rank generates only its rows; reference group table per shard
        k, x, y, z, w = G.c3_tables(300_001, 3, part=(rank, world), slicer=slicer)
        ks, vs, _ = ref.group_aggregate([k], [x, k, z], ["sum", "count", "sum"])
        out["c3"] = O.Partial([ks[0]], [vs[0], vs[1], vs[2]])
        # Q1 shard: group tables in partial form (sums + count)
        t = Q.lineitem_q1(200_000, 43, part=(rank, world), slicer=slicer)
        api = refpy.RefAPI(ref)
        C_, A_ = api.compute, api.agg
        msk = C_.compare_scalar(t["l_shipdate"], Q.Q1_CUTOFF, "<=")
        f = {n: C_.filter(v, msk) for n, v in t.items()}
        ks, vs, _ = A_.group_aggregate([f["l_returnflag"], f["l_linestatus"]],
                                       [f["l_quantity"], f["l_quantity"]], ["sum", "count"], normalize=True)
        out["q1"] = O.Partial(ks, vs)
        gathered = [None] * world
        dist.all_gather_object(gathered, out)
        if rank == 0:
            q.put(gathered)
    finally:
        dist.destroy_process_group()


def test_two_rank_shard_and_merge(ref):
    from oracle import streaming as O
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a, b, c = G.c2_tables(400_000, seed=11)
    m = ref.compare_scalar(c, 20, "<")
    want = ref.aggregate_all(ref.arith(ref.filter(a, m), ref.filter(b, m), "*"), "sum")
    tot = int(np.array([g["c2"] for g in gathered], np.int64).astype(np.uint64).sum().astype(np.int64))
    assert tot == want
    k, x, y, z, w = G.c3_tables(300_001, 3)
    wk, wv, _ = ref.group_aggregate([k], [x, k, z], ["sum", "count", "avg"])
    mg = O.merge([g["c3"] for g in gathered])
    assert np.array_equal(mg.keys[0], wk[0])
    assert np.array_equal(mg.parts[0], wv[0]) and np.array_equal(mg.parts[1], wv[1])
    assert np.array_equal(mg.parts[2] / mg.parts[1], wv[2])  # AVG from merged SUM / COUNT, never averaged
    from oracle.refpy import RefAPI
    ks, vs, _ = Q.q1(RefAPI(ref), Q.lineitem_q1(200_000, 43))
    mq = O.merge([g["q1"] for g in gathered])
    assert all(np.array_equal(a_, b_) for a_, b_ in zip(mq.keys, ks))
    assert np.array_equal(mq.parts[0], vs[0]) and np.array_equal(mq.parts[1], vs[7])


def test_plan_cuts_snap():
    a = G.gapless_rle(10_000, 64, 1)
    cuts = S.plan_cuts(10_000, 4, a)
    assert cuts[0] == 0 and cuts[-1] == 10_000 and len(cuts) == 5
    ends = set((a.e + 1).tolist())
    assert all(c in ends for c in cuts[1:-1])
