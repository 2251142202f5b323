"""Row-range sharding and partial-aggregate merge.

The path partitions by row range: every rank owns rows [lo, hi) of each
column as a standalone shard (``rq_shard_host_column``: runs crossing a cut
are split with the value duplicated, positions rebased, total = hi − lo), so
per-rank execution needs no data exchange. Results combine with ONE
collective:

* global aggregates: int64 SUM / COUNT add with wrap-around (the reference's
  int64 accumulators, groupby.cpp:82-89), f64 SUM adds (1e-9 relative),
  MIN / MAX fold, AVG is recomputed from the merged SUM and COUNT — never
  averaged;
* dense group tables (dictionary-code slots): slot-wise add of (sum, count),
  presence = count > 0, keys re-derived in ascending order.

Host-only module: importable and testable without a GPU (the C-ABI library's
``rq_shard_host_column`` is a pure host function).
"""
from __future__ import annotations

from typing import Dict, List, Sequence

import numpy as np

from . import host as H


def plan_cuts(total: int, world: int, snap_to: H.RleColumn = None) -> List[int]:
    """Cut points p_g = floor(g·N/G), optionally snapped to the nearest run
    boundary of ``snap_to`` so the column with the most runs is never split."""
    cuts = [total * g // world for g in range(world + 1)]
    if snap_to is not None and len(snap_to.e) > 0:
        ends = snap_to.e
        for g in range(1, world):
            i = int(np.searchsorted(ends, cuts[g] - 1))
            if i < len(ends):
                cuts[g] = int(ends[i]) + 1
        cuts = sorted(set(min(max(c, 0), total) for c in cuts))
        while len(cuts) < world + 1:  # degenerate: fewer runs than ranks
            cuts.append(total)
    return cuts


def shard_table(columns: Dict[str, H.Column], rank: int, world: int, snap: str = None) -> Dict[str, H.Column]:
    """This rank's shard of every column (same row range for all columns)."""
    from .runq import shard_host_column
    total = next(iter(columns.values())).total_size
    cuts = plan_cuts(total, world, columns.get(snap) if snap else None)
    lo, hi = cuts[rank], cuts[rank + 1]
    return {k: shard_host_column(c, lo, hi) for k, c in columns.items()}


def wrap_i64(x: int) -> int:
    return int(np.array(x, dtype=np.uint64).astype(np.int64)) if x >= 0 else int(np.int64(x))


def merge_scalar(partials: Sequence, fn: str, counts: Sequence[int] = None):
    """Combine per-shard aggregate results. AVG needs (sum, count) partials:
    pass the partial SUMs and ``counts``."""
    if fn in ("sum", "count"):
        if any(isinstance(p, float) for p in partials):
            return float(sum(partials))
        acc = np.uint64(0)
        for p in partials:
            acc = acc + np.array(p, dtype=np.int64).astype(np.uint64)  # wraps mod 2^64
        return int(acc.astype(np.int64))
    if fn == "min":
        return min(partials)
    if fn == "max":
        return max(partials)
    if fn == "avg":
        n = sum(counts)
        return float(sum(partials)) / n if n else float("nan")
    raise ValueError(fn)


def merge_group_tables(keys: Sequence[np.ndarray], sums: Sequence[np.ndarray],
                       counts: Sequence[np.ndarray]):
    """Merge per-shard group-by results (ascending keys, SUM, COUNT per key)
    into the global table: keys ascending, SUM added (int wraps), COUNT
    added; AVG = SUM / COUNT recomputed by the caller."""
    allk = np.concatenate(keys)
    uk, inv = np.unique(allk, return_inverse=True)
    sdt = np.result_type(*[s.dtype for s in sums]) if sums else np.int64
    out_s = np.zeros(len(uk), dtype=sdt)
    out_c = np.zeros(len(uk), dtype=np.int64)
    off = 0
    for k, s, c in zip(keys, sums, counts):
        idx = inv[off:off + len(k)]
        np.add.at(out_s, idx, s)
        np.add.at(out_c, idx, c)
        off += len(k)
    return uk, out_s, out_c


def allreduce_scalar_i64(value: int, group=None) -> int:
    """One NCCL/gloo all_reduce of an int64 partial (wrapping sum)."""
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([value], dtype=torch.int64, device=dev)
    dist.all_reduce(t, group=group)
    return int(t.item())
