"""ctypes loader for libms.so (the C ABI declared in include/multisplit.h).

Argument marshalling only.  There is no CPU fallback: if the shared library
is missing or fails to load, every call raises.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libms.so")

MS_SUCCESS = 0
MS_ERR_INVALID_VALUE = 1
MS_ERR_UNSUPPORTED = 2
MS_ERR_WORKSPACE = 3
MS_ERR_CUDA = 4
MS_ERR_KEY_DOMAIN = 5
MS_ERR_NCCL = 6

MS_OPT_RANK = 0
MS_OPT_RUN_STORES = 1
MS_OPT_PIPELINE = 2
MS_OPT_SORT = 3
MS_RANK_AUTO = 0
MS_RANK_PEER_MASKS = 1
MS_PIPELINE_LEVEL0 = 0
MS_PIPELINE_TILE = 1
MS_PIPELINE_ONESWEEP = 2
MS_PIPELINE_AUTO = 3
MS_SORT_AUTO = 0
MS_SORT_PASSES = 1

MS_BUCKET_IDENTITY = 0
MS_BUCKET_DELTA = 1
MS_BUCKET_RADIX = 2
MS_BUCKET_SPLITTERS = 3


class ms_sssp_stats(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_uint64), ("items", ctypes.c_uint64),
                ("frontier", ctypes.c_uint64), ("pushes", ctypes.c_uint64)]


class ms_bucket_fn(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_uint32), ("num_buckets", ctypes.c_uint32),
                ("delta", ctypes.c_uint32), ("shift", ctypes.c_uint32), ("bits", ctypes.c_uint32),
                ("splitters", ctypes.c_void_p)]


# (name, restype, argtypes) for every symbol include/multisplit.h declares.
_P, _U32, _U64, _SZ, _I = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_size_t, ctypes.c_int
_FN = ctypes.POINTER(ms_bucket_fn)
_U32P = ctypes.POINTER(ctypes.c_uint32)
SIGNATURES = [
    ("ms_status_string", ctypes.c_char_p, [_I]),
    ("ms_version", ctypes.c_char_p, []),
    ("ms_lane_ordered_increment", _I, []),
    ("ms_device_init", _I, [_I]),
    ("ms_set_option", _I, [_I, _I]),
    ("ms_get_option", _I, [_I]),
    ("ms_bucket_delta_default", _I, [_U32, _FN]),
    ("ms_bucket_identity", _I, [_U32, _FN]),
    ("ms_bucket_radix", _I, [_U32, _U32, _FN]),
    ("ms_bucket_validate", _I, [_FN]),
    ("ms_multisplit_workspace_size", _SZ, [_U64, _U32, _I]),
    ("ms_multisplit_keys", _I, [_P, _P, _U64, _FN, _P, _P, _SZ, _P]),
    ("ms_multisplit_pairs", _I, [_P, _P, _P, _P, _U64, _FN, _P, _P, _SZ, _P]),
    ("ms_radix_sort_workspace_size", _SZ, [_U64, _I]),
    ("ms_radix_sort_keys", _I, [_P, _P, _U64, _U32, _U32, _U32, _P, _SZ, _P]),
    ("ms_radix_sort_pairs", _I, [_P, _P, _P, _P, _U64, _U32, _U32, _U32, _P, _SZ, _P]),
    ("ms_radix_pass_schedule", _I, [_U32, _U32, _U32, _U32P, _U32P, _I]),
    ("ms_device_status", _I, [_P, _P]),
    ("ms_multisplit_tile_size", _U32, [_U32, _I]),
    ("ms_stage_prescan", _I, [_P, _U64, _FN, _P, _U32, _P]),
    ("ms_stage_scan_workspace_size", _SZ, [_U64, _U32]),
    ("ms_stage_scan", _I, [_P, _P, _U64, _U32, _P, _P, _SZ, _P]),
    ("ms_shard_plan", _I, [_P, _U32, _U32, _U32, _P, _P, _P, _P, _P, _P]),
    ("ms_shard_merge_keys", _I, [_P, _U64, _FN, _P, _P, _U32, _P, _P]),
    ("ms_shard_merge_pairs", _I, [_P, _P, _U64, _FN, _P, _P, _U32, _P, _P, _P]),
    ("ms_histogram_even", _I, [_P, _U64, _U32, ctypes.c_float, ctypes.c_float, _P, _P]),
    ("ms_histogram_range", _I, [_P, _U64, _U32, _P, _P, _P]),
    ("ms_comm_unique_id", _I, [_P]),
    ("ms_comm_init", _I, [ctypes.POINTER(ctypes.c_void_p), _I, _I, _P, _I]),
    ("ms_comm_destroy", _I, [_P]),
    ("ms_comm_check", _I, [_P]),
    ("ms_comm_abort", _I, [_P]),
    ("ms_comm_register_output", _I, [_P, _P, _P, _U64]),
    ("ms_sharded_workspace_size", _SZ, [_P, _U64, _U32, _I]),
    ("ms_multisplit_keys_sharded", _I, [_P, _P, _P, _U64, _FN, _P, _P, _SZ, _P]),
    ("ms_multisplit_pairs_sharded", _I, [_P, _P, _P, _P, _P, _U64, _FN, _P, _P, _SZ, _P]),
    ("ms_shard_workspace_size", _SZ, [_U64, _U32, _U32, _I]),
    ("ms_shard_prescan", _I, [_P, _U64, _FN, _I, _U32, _P, _P, _SZ, _P]),
    ("ms_shard_scatter", _I, [_P, _P, _U64, _FN, _P, _U32, _U32, _P, _P, _P, _P, _SZ, _P]),
    ("ms_sssp_workspace_size", _SZ, [_U32, _U64, _U32]),
    ("ms_sssp", _I, [_P, _P, _P, _U32, _U64, _U32, _U32, _U32, _P, _P, _SZ, _P, _P]),
    ("ms_set_stage_events", None, [_P]),
    ("ms_launch_count", _U64, []),
]

_lib = None


def load() -> ctypes.CDLL:
    """Load libms.so (built by __graft_entry__.build()); raise if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _lib = lib
    return _lib


class MultisplitError(RuntimeError):
    def __init__(self, code: int, where: str = ""):
        name = load().ms_status_string(code).decode()
        super().__init__(f"{where}: {name} ({code})" if where else f"{name} ({code})")
        self.code = code


def check(code: int, where: str = "") -> None:
    if code != MS_SUCCESS:
        raise MultisplitError(code, where)
