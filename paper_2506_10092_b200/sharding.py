"""Row-range sharding and partial-aggregate merge.

The path partitions by row range: every rank owns rows [lo, hi) of each
column as a standalone shard (``rq_shard_host_column``: runs crossing a cut
are split with the value duplicated, positions rebased, total = hi − lo), so
per-rank execution needs no data exchange. Results combine with ONE
collective inside the library (csrc/comm.cu, ``rq_*_sharded``): a grouped
NCCL all-reduce of the global partials, or an all-gather of the (key,
partial) group tables regrouped on the device; AVG recomputed from the
merged SUM and COUNT.

Host-only module: importable and testable without a GPU (the C-ABI library's
``rq_shard_host_column`` is a pure host function).
"""
from __future__ import annotations

from typing import Dict, List

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
