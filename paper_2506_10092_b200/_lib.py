"""Loader and ctypes prototypes for the in-tree C ABI library.

``librunq_b200.so`` is built in-tree by ``__graft_entry__.build()``
(``paper_2506_10092_b200/csrc/Makefile``). There is no fallback: if the
library is missing or a symbol is absent, importing the device API raises.
"""
from __future__ import annotations

import ctypes as C
import os

from .host import ColumnStats, EncodingChoice, Expr, Heuristic, HostColumn, HostMask, JoinSide, Pred, Scalar

LIB_PATH = os.environ.get("RQ_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "librunq_b200.so")

_lib = None

vp = C.c_void_p
i32 = C.c_int32
i64 = C.c_int64
P = C.POINTER

# name -> (restype, argtypes). Mirrors include/runq_b200.h one to one.
PROTOTYPES = {
    "rq_last_error": (C.c_char_p, []),
    "rq_version": (C.c_char_p, []),
    "rq_ctx_create": (C.c_int, [C.c_int, P(vp)]),
    "rq_ctx_destroy": (C.c_int, [vp]),
    "rq_ctx_synchronize": (C.c_int, [vp]),
    "rq_ctx_stream": (vp, [vp]),
    "rq_ctx_launches": (i64, [vp]),
    "rq_ctx_set_profiling": (C.c_int, [vp, i32]),
    "rq_ctx_profile_only": (C.c_int, [vp, C.c_char_p]),
    "rq_ctx_profile_report": (C.c_int, [vp, i32, C.c_char_p, i64]),
    "rq_arr_upload": (C.c_int, [vp, i32, vp, i64, P(vp)]),
    "rq_arr_wrap_device": (C.c_int, [vp, i32, vp, i64, P(vp)]),
    "rq_arr_alloc": (C.c_int, [vp, i32, i64, P(vp)]),
    "rq_arr_write": (C.c_int, [vp, vp, i64, vp, i64]),
    "rq_arr_info": (C.c_int, [vp, P(i32), P(i64)]),
    "rq_arr_device_ptr": (vp, [vp]),
    "rq_arr_download": (C.c_int, [vp, vp, vp]),
    "rq_arr_download_many": (C.c_int, [vp, i32, P(vp), P(vp)]),
    "rq_arr_free": (C.c_int, [vp]),
    "rq_col_upload": (C.c_int, [vp, P(HostColumn), P(vp)]),
    "rq_col_describe": (C.c_int, [vp, P(HostColumn)]),
    "rq_col_download": (C.c_int, [vp, vp, P(HostColumn)]),
    "rq_col_dump_image": (C.c_int, [vp, vp, P(vp), P(C.c_int64)]),
    "rq_col_load_image": (C.c_int, [vp, vp, C.c_int64, P(vp)]),
    "rq_image_free": (None, [vp]),
    "rq_col_free": (C.c_int, [vp]),
    "rq_col_encoding": (C.c_int, [vp]),
    "rq_col_total_size": (i64, [vp]),
    "rq_col_value_type": (C.c_int, [vp]),
    "rq_col_make_rle": (C.c_int, [vp, vp, vp, vp, i64, P(vp)]),
    "rq_col_make_index": (C.c_int, [vp, vp, vp, i64, P(vp)]),
    "rq_col_make_plain": (C.c_int, [vp, vp, i32, i32, i64, P(vp)]),
    "rq_col_part": (C.c_int, [vp, C.c_int, P(vp)]),
    "rq_mask_upload": (C.c_int, [vp, P(HostMask), P(vp)]),
    "rq_mask_describe": (C.c_int, [vp, P(HostMask)]),
    "rq_mask_download": (C.c_int, [vp, vp, P(HostMask)]),
    "rq_mask_free": (C.c_int, [vp]),
    "rq_mask_true_count": (C.c_int, [vp, vp, P(i64)]),
    "rq_range_intersect": (C.c_int, [vp, vp, vp, vp, vp, P(vp), P(vp), P(vp), P(vp)]),
    "rq_idx_in_rle": (C.c_int, [vp, vp, vp, vp, P(vp), P(vp), P(vp)]),
    "rq_rle_contain_idx": (C.c_int, [vp, vp, vp, vp, P(vp), P(vp), P(vp)]),
    "rq_idx_in_idx": (C.c_int, [vp, vp, vp, P(vp), P(vp), P(vp)]),
    "rq_plain_mask_to_rle": (C.c_int, [vp, vp, P(vp)]),
    "rq_plain_mask_to_index": (C.c_int, [vp, vp, P(vp)]),
    "rq_compact_rle": (C.c_int, [vp, vp, P(vp)]),
    "rq_plain_to_rle": (C.c_int, [vp, vp, P(vp)]),
    "rq_plain_to_rle_index": (C.c_int, [vp, vp, C.c_int64, P(vp)]),
    "rq_plain_to_plain_index": (C.c_int, [vp, vp, C.c_double, P(vp)]),
    "rq_heuristic_default": (None, [P(Heuristic)]),
    "rq_choose_encoding": (C.c_int, [vp, vp, P(Heuristic), P(EncodingChoice)]),
    "rq_encode": (C.c_int, [vp, vp, P(EncodingChoice), P(vp)]),
    "rq_sort_table": (C.c_int, [vp, P(vp), i32, P(i32), i32, P(vp)]),
    "rq_bucketize": (C.c_int, [vp, vp, vp, i32, P(vp)]),
    "rq_decode_values": (C.c_int, [vp, vp, P(vp)]),
    "rq_normalize_basic": (C.c_int, [vp, vp, P(vp)]),
    "rq_align": (C.c_int, [vp, vp, vp, P(i32), P(vp), P(vp), P(vp), P(vp), P(vp)]),
    "rq_arith": (C.c_int, [vp, vp, vp, i32, P(vp)]),
    "rq_compare": (C.c_int, [vp, vp, vp, i32, P(vp)]),
    "rq_arith_scalar": (C.c_int, [vp, vp, Scalar, i32, i32, P(vp)]),
    "rq_compare_scalar": (C.c_int, [vp, vp, Scalar, i32, i32, P(vp)]),
    "rq_filter": (C.c_int, [vp, vp, vp, P(vp)]),
    "rq_mask_and": (C.c_int, [vp, vp, vp, P(vp)]),
    "rq_mask_or": (C.c_int, [vp, vp, vp, P(vp)]),
    "rq_mask_not": (C.c_int, [vp, vp, P(vp)]),
    "rq_aggregate_all": (C.c_int, [vp, vp, i32, P(i32), P(i64), P(C.c_double)]),
    "rq_group_aggregate": (C.c_int, [vp, P(vp), i32, P(vp), P(i32), i32, P(i64), P(vp), P(vp)]),
    "rq_group_aggregate_normalized": (C.c_int, [vp, P(vp), i32, P(vp), P(i32), i32, P(i64), P(vp), P(vp)]),
    "rq_aggregate_binop": (C.c_int, [vp, vp, vp, i32, i32, P(i32), P(i64), P(C.c_double)]),
    "rq_filtered_aggregate_binop": (C.c_int, [vp, vp, Scalar, i32, vp, vp, i32, i32, P(i32), P(i64),
                                              P(C.c_double)]),
    "rq_group_aggregate_exprs": (C.c_int, [vp, vp, P(vp), i32, P(Expr), P(i32), i32, P(i64), P(vp), P(vp),
                                           P(i32)]),
    "rq_group_aggregate_where": (C.c_int, [vp, P(Pred), i32, vp, P(vp), i32, P(Expr), P(i32), i32, P(i64), P(vp),
                                           P(vp), P(i32)]),
    "rq_semi_join_mask": (C.c_int, [vp, vp, vp, P(vp)]),
    "rq_hash_build_probe": (C.c_int, [vp, vp, vp, P(vp), P(vp)]),
    "rq_get_join_index": (C.c_int, [vp, vp, vp, P(JoinSide), P(JoinSide), P(i64)]),
    "rq_apply_join_index": (C.c_int, [vp, vp, P(JoinSide), P(vp)]),
    "rq_catalog_create": (C.c_int, [P(vp)]),
    "rq_catalog_destroy": (C.c_int, [vp]),
    "rq_catalog_add_column": (C.c_int, [vp, C.c_char_p, C.c_char_p, vp, P(C.c_char_p), i64, C.c_char_p, i32]),
    "rq_run_plan": (C.c_int, [vp, vp, C.c_char_p, P(vp)]),
    "rq_result_info": (C.c_int, [vp, P(i32), P(i64), P(i32)]),
    "rq_result_column": (C.c_int, [vp, i32, P(C.c_char_p), P(vp)]),
    "rq_result_free": (C.c_int, [vp]),
    "rq_shard_host_column": (C.c_int, [P(HostColumn), i64, i64, P(HostColumn)]),
    "rq_host_column_free": (None, [P(HostColumn)]),
    "rq_comm_unique_id": (C.c_int, [vp, i64]),
    "rq_comm_init_nccl": (C.c_int, [vp, vp, i32, i32, P(vp)]),
    "rq_comm_init_host": (C.c_int, [vp, i32, i32, vp, vp, P(vp)]),
    "rq_comm_info": (C.c_int, [vp, P(i32), P(i32), P(i32)]),
    "rq_comm_destroy": (C.c_int, [vp]),
    "rq_merge_group_tables": (C.c_int, [vp, vp, P(vp), i32, P(vp), P(i32), i32, i64, P(i64), P(vp), P(vp)]),
    "rq_aggregate_all_sharded": (C.c_int, [vp, vp, vp, i32, P(i32), P(i64), P(C.c_double)]),
    "rq_aggregate_binop_sharded": (C.c_int, [vp, vp, vp, vp, i32, i32, P(i32), P(i64), P(C.c_double)]),
    "rq_filtered_aggregate_binop_sharded": (C.c_int, [vp, vp, vp, Scalar, i32, vp, vp, i32, i32, P(i32), P(i64),
                                                      P(C.c_double)]),
    "rq_group_aggregate_sharded": (C.c_int, [vp, vp, P(vp), i32, P(vp), P(i32), i32, i32, P(i64), P(vp), P(vp)]),
    "rq_group_aggregate_where_sharded": (C.c_int, [vp, vp, vp, i32, vp, P(vp), i32, vp, P(i32), i32, P(i64), P(vp),
                                                   P(vp), P(i32)]),
    "rq_decompose": (C.c_int, [vp, vp, P(i32), P(i64), P(vp), P(vp), P(vp), P(vp)]),
    "rq_align_many": (C.c_int, [vp, P(vp), i32, P(i32), P(i64), P(vp), P(vp), P(vp), P(vp)]),
    "rq_shape_weights": (C.c_int, [vp, i32, i64, vp, vp, vp, P(vp)]),
    "rq_group": (C.c_int, [vp, P(vp), i32, P(i32), P(i64), P(vp), P(vp), P(vp), P(vp), P(vp), P(i64)]),
    "rq_group_on_arrays": (C.c_int, [vp, P(vp), i32, P(vp), P(vp), P(i64)]),
    "rq_aggregate_array": (C.c_int, [vp, i32, i64, vp, vp, vp, vp, vp, i64, i32, P(vp)]),
    "rq_scatter_reduce": (C.c_int, [vp, vp, vp, i64, i32, P(vp)]),
    "rq_unique_with_inverse": (C.c_int, [vp, P(vp), i32, P(vp), P(vp), P(i64)]),
    "rq_cumsum": (C.c_int, [vp, vp, i32, P(vp)]),
    "rq_checked_sum": (C.c_int, [vp, vp, P(i64)]),
    "rq_repeat_interleave": (C.c_int, [vp, vp, vp, P(vp)]),
    "rq_range_arange": (C.c_int, [vp, vp, vp, P(vp)]),
    "rq_gather": (C.c_int, [vp, vp, vp, P(vp)]),
    "rq_sort_with_perm": (C.c_int, [vp, vp, P(vp), P(vp)]),
    "rq_adjacent_ne": (C.c_int, [vp, vp, P(vp)]),
    "rq_range_union": (C.c_int, [vp, vp, vp, vp, vp, P(vp), P(vp)]),
    "rq_merge_sorted_idx": (C.c_int, [vp, vp, vp, P(vp)]),
    "rq_concat_sort_idx": (C.c_int, [vp, vp, vp, P(vp)]),
    "rq_complement_rle": (C.c_int, [vp, vp, vp, i64, P(vp), P(vp)]),
    "rq_complement_index": (C.c_int, [vp, vp, i64, P(vp), P(vp)]),
    "rq_rle_to_index": (C.c_int, [vp, vp, i64, P(vp)]),
    "rq_rle_to_plain": (C.c_int, [vp, vp, C.c_double, i64, P(vp)]),
    "rq_mask_rle_to_index": (C.c_int, [vp, vp, i64, P(vp)]),
    "rq_mask_rle_to_plain": (C.c_int, [vp, vp, i64, P(vp)]),
    "rq_compact_rle_index": (C.c_int, [vp, vp, P(vp)]),
    "rq_decode_full": (C.c_int, [vp, vp, P(vp)]),
    "rq_to_rows": (C.c_int, [vp, vp, P(vp), P(vp)]),
    "rq_col_stats": (C.c_int, [vp, vp, P(ColumnStats)]),
}

# host-transport all-gather callback (include/runq_b200.h rq_host_allgather_fn)
HOST_ALLGATHER_FN = C.CFUNCTYPE(C.c_int, vp, i64, vp, vp)


class RqError(RuntimeError):
    """runq::Error (error.hpp:11-14)."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class RqOverflowError(RqError):
    """runq::OverflowError (error.hpp:17-20)."""


class RqResourceError(RqError):
    """runq::ResourceError (error.hpp:23-26)."""


class RqDeviceError(RqError):
    """CUDA / NCCL failure."""


def load():
    """Loads the library (once). Raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} not found: the CUDA extension is not built (run __graft_entry__.build()); "
            "there is no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in PROTOTYPES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status: int):
    if status == 0:
        return
    msg = load().rq_last_error().decode(errors="replace")
    if status == 2:
        raise RqOverflowError(status, msg)
    if status == 3:
        raise RqResourceError(status, msg)
    if status in (4, 5):
        raise RqDeviceError(status, msg)
    raise RqError(status, msg)
