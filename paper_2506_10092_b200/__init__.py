"""B200-native compressed-execution query path of arXiv 2506.10092 (`runq`).

Layout:
  csrc/            sm_100a CUDA kernels + C++ host dispatch + the C ABI
                   (include/runq_b200.h), built in-tree to librunq_b200.so
  host.py          host column images mirroring runq's column model (no GPU)
  runq.py          the reference operator API over the C ABI (device path)
  sharding.py      row-range shard planner + partial-aggregate merge (multi-GPU)

``import paper_2506_10092_b200.runq`` loads the CUDA library and raises if it
is missing; ``host`` and ``sharding`` are importable without it.
"""
from . import host  # noqa: F401

__all__ = ["host"]
