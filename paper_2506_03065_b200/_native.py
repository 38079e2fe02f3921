"""ctypes binding of the C ABI declared in include/svdit_b200.h.

The product path has no Python or CPU fallback: if the native library is
missing or fails to load, every call raises immediately.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_int32, c_int64, c_uint8, c_void_p
from pathlib import Path

import numpy as np

from .errors import (
    ConfigError,
    DegenerateMaskError,
    DegenerateRowError,
    ShapeError,
    SvditError,
)

LIB_PATH = Path(os.environ.get("SVD_LIB", Path(__file__).resolve().parent / "libsvdit_b200.so"))

SVD_OK = 0
_STATUS_TO_EXC = {
    1: ShapeError,
    2: DegenerateRowError,
    3: DegenerateMaskError,
    4: ConfigError,
}


class NativeError(SvditError, RuntimeError):
    """CUDA failure or a shape the sm_100a kernel does not support."""


class SvdLayout(ctypes.Structure):
    _fields_ = [
        ("text_tokens", c_int64),
        ("frames", c_int64),
        ("tokens_per_frame", c_int64),
        ("block_size", c_int64),
    ]


class SvdSpec(ctypes.Structure):
    _fields_ = [
        ("mode", c_int32),
        ("halfwidth", c_int32),
        ("period", c_int32),
        ("md_halfwidth", c_int32),
        ("stripe_count", c_int32),
        ("include_diagonal", c_int32),
        ("n_stripes", c_int32),
        ("stripes", POINTER(c_int64)),
    ]


class SvdPlanInfo(ctypes.Structure):
    _fields_ = [
        ("n_tokens", c_int64),
        ("n_blocks", c_int64),
        ("n_segments", c_int64),
        ("n_heads", c_int32),
        ("n_groups", c_int32),
        ("fine_mask", c_int32),
        ("sharded", c_int32),
        ("n_work_items", c_int64),
        ("n_kv_entries", c_int64),
        ("computed_tiles", c_int64),
        ("active_pairs", c_double),
        ("dense_pairs", c_double),
        ("n_split_groups", c_int32),
        ("max_split_parts", c_int32),
    ]


class SvdFwdArgs(ctypes.Structure):
    """include/svdit_b200.h svd_fwd_args."""

    _fields_ = [
        ("q", c_void_p), ("k", c_void_p), ("v", c_void_p), ("o", c_void_p),
        ("q_strides", c_int64 * 4), ("k_strides", c_int64 * 4), ("v_strides", c_int64 * 4),
        ("o_strides", c_int64 * 4),
        ("batch", c_int32), ("head_dim", c_int32), ("tensor_dim", c_int32), ("dtype", c_int32),
        ("in_heads", c_int32), ("stats_heads", c_int32),
        ("in_head_map", c_void_p), ("o_head_map", c_void_p), ("nonfinite", c_void_p),
        ("row_stats", c_void_p),
    ]


# every exported symbol with its signature (restype, argtypes)
SIGNATURES = {
    "svd_last_error": (c_char_p, []),
    "svd_version": (c_char_p, []),
    "svd_grid_size": (c_int, [POINTER(SvdLayout), POINTER(c_int64), POINTER(c_int64)]),
    "svd_grid_arrays": (c_int, [POINTER(SvdLayout), c_void_p, c_void_p, c_void_p, c_void_p]),
    "svd_frame_period": (c_int, [POINTER(SvdLayout), POINTER(c_int64)]),
    "svd_mask_build": (c_int, [POINTER(SvdLayout), POINTER(SvdSpec), c_void_p, POINTER(c_int32)]),
    "svd_plan_create": (c_int, [POINTER(SvdLayout), POINTER(SvdSpec), c_int32, POINTER(c_void_p)]),
    "svd_plan_create_from_masks": (
        c_int,
        [POINTER(SvdLayout), c_int32, c_void_p, c_void_p, c_void_p, c_int32, POINTER(c_void_p)],
    ),
    "svd_plan_destroy": (None, [c_void_p]),
    "svd_plan_get_info": (c_int, [c_void_p, POINTER(SvdPlanInfo)]),
    "svd_plan_group_heads": (c_int, [c_void_p, c_int32, c_void_p, POINTER(c_int32), POINTER(c_int32)]),
    "svd_plan_group_mask": (c_int, [c_void_p, c_int32, c_void_p]),
    "svd_plan_group_nnz": (c_int, [c_void_p, c_int32, POINTER(c_int64)]),
    "svd_plan_group_csr": (c_int, [c_void_p, c_int32, c_void_p, c_void_p]),
    "svd_plan_schedule": (c_int, [c_void_p, c_void_p, c_void_p]),
    "svd_plan_subset": (c_int, [c_void_p, c_void_p, c_int32, POINTER(c_void_p)]),
    "svd_plan_shard": (c_int, [c_void_p, c_int32, c_int32, POINTER(c_void_p)]),
    "svd_plan_shard_sm": (c_int, [c_void_p, c_int32, c_int32, c_int32, c_int32, POINTER(c_void_p)]),
    "svd_plan_shard_ex": (c_int, [c_void_p, c_int32, c_int32, c_int32, c_int32, c_int32, POINTER(c_void_p)]),
    "svd_plan_shard_rows": (c_int, [c_void_p, POINTER(c_int64), c_void_p, c_void_p]),
    "svd_plan_shard_heads": (c_int, [c_void_p, c_void_p, c_int32, POINTER(c_void_p)]),
    "svd_attn_fwd": (
        c_int,
        [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
         POINTER(c_int64), POINTER(c_int64), POINTER(c_int64), POINTER(c_int64),
         c_int32, c_int32, c_int32, c_int32, c_void_p],
    ),
    "svd_attn_fwd_ex": (
        c_int,
        [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
         POINTER(c_int64), POINTER(c_int64), POINTER(c_int64), POINTER(c_int64),
         c_int32, c_int32, c_int32, c_int32, c_void_p, c_void_p],
    ),
    "svd_attn_fwd_v2": (
        c_int,
        [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
         POINTER(c_int64), POINTER(c_int64), POINTER(c_int64), POINTER(c_int64),
         c_int32, c_int32, c_int32, c_int32, c_void_p, c_void_p, c_void_p],
    ),
    "svd_attn_fwd_args": (c_int, [c_void_p, POINTER(SvdFwdArgs), c_void_p]),
    "svd_block_key_mass_from_stats": (
        c_int,
        [c_void_p, c_void_p, POINTER(c_int64), POINTER(c_int64), c_int32, c_int32, c_int64, c_int32,
         c_int32, c_int32, c_int32, c_void_p, c_void_p, c_int64, c_void_p, c_void_p],
    ),
    "svd_attn_fwd_peers": (
        c_int,
        [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int32,
         POINTER(c_int64), POINTER(c_int64), POINTER(c_int64), POINTER(c_int64),
         c_int32, c_int32, c_int32, c_int32, c_void_p],
    ),
    "svd_peer_barrier": (c_int, [c_void_p, c_int32, c_int32, c_int32, c_void_p, c_double, c_void_p]),
    "svd_ipc_export": (c_int, [c_void_p, c_void_p, POINTER(c_int64)]),
    "svd_ipc_import": (c_int, [c_void_p, c_int64, POINTER(c_void_p)]),
    "svd_ipc_close": (c_int, [c_void_p, c_int64]),
    "svd_head_sqdiff": (
        c_int,
        [c_void_p, c_void_p, POINTER(c_int64), POINTER(c_int64), c_int32, c_int32, c_int64, c_int32,
         c_void_p, c_void_p],
    ),
    "svd_unpack_rows": (
        c_int,
        [c_void_p, c_void_p, c_int64, c_void_p, c_int64, c_void_p, POINTER(c_int64), c_int32, c_void_p],
    ),
    "svd_key_mass_workspace": (c_int64, [c_int32, c_int32, c_int64]),
    "svd_block_key_mass": (
        c_int,
        [c_void_p, c_void_p, POINTER(c_int64), POINTER(c_int64), c_int32, c_int32, c_int64, c_int32,
         c_int32, c_int32, c_int32, c_void_p, c_int64, c_void_p, c_void_p],
    ),
    "svd_layernorm": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int32, ctypes.c_float,
                              c_void_p]),
    "svd_rope_table": (c_int, [c_void_p, c_int64, c_int32, c_double, c_void_p]),
    "svd_rope_apply": (c_int, [c_void_p, c_int64, c_int64, c_int64, c_int64, c_int32, c_int32, c_void_p,
                               c_void_p]),
    "svd_gelu": (c_int, [c_void_p, c_int64, c_void_p]),
    "svd_gemm": (c_int, [c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64, c_int64, c_int64, c_int64,
                         c_int32, c_void_p, c_int64, c_void_p, c_int32, c_int32, c_int64, c_void_p]),
}

_lib = None


def lib() -> ctypes.CDLL:
    """Load (once) the in-tree native library; raise loudly if it is absent."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise NativeError(
                f"native library {LIB_PATH} not built: run "
                "`python -m paper_2506_03065_b200._build` (or __graft_entry__.build())"
            )
        handle = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(status: int) -> None:
    if status == SVD_OK:
        return
    msg = lib().svd_last_error().decode("utf-8", "replace")
    exc = _STATUS_TO_EXC.get(status, NativeError)
    raise exc(msg)


def make_layout(layout) -> SvdLayout:
    return SvdLayout(int(layout.text_tokens), int(layout.frames), int(layout.tokens_per_frame),
                     int(layout.block_size))


def make_spec(spec, keep: list) -> SvdSpec:
    """Encode a PatternSpec.  `keep` holds buffers that must outlive the call."""
    if spec.stripes is None:
        n, ptr = -1, None
    else:
        arr = np.ascontiguousarray(np.asarray(spec.stripes, dtype=np.int64))
        keep.append(arr)
        n, ptr = int(arr.size), arr.ctypes.data_as(POINTER(c_int64))
    return SvdSpec(
        int(spec.mode),
        int(spec.halfwidth),
        int(spec.period) if spec.period is not None else -1,
        int(spec.md_halfwidth),
        int(spec.stripe_count),
        1 if spec.include_diagonal else 0,
        n,
        ptr,
    )


def ptr(arr: np.ndarray) -> c_void_p:
    return c_void_p(arr.ctypes.data)


def i64x4(values) -> ctypes.Array:
    return (c_int64 * 4)(*[int(v) for v in values])


__all__ = [
    "NativeError", "SvdLayout", "SvdSpec", "SvdPlanInfo", "SIGNATURES", "LIB_PATH",
    "lib", "check", "make_layout", "make_spec", "ptr", "i64x4", "c_int32", "c_int64",
    "c_uint8", "c_void_p",
]
