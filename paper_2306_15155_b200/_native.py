"""ctypes binding of ``lib/libgnnc.so`` (C ABI: ``include/gnnc.h``).

There is no CPU fallback: every compute entry point requires CUDA tensors and
raises if the library or the device is missing.  Host-only entry points
(planner, partitioner, version/launch counters) work without a GPU.
"""

from __future__ import annotations

import ctypes
import os
import re
from pathlib import Path

from ._build import LIB, ROOT

ABI_VERSION = 2  # GNNC_ABI_VERSION of include/gnnc.h
GC_RELU = 1 << 0
GC_ACCUMULATE = 1 << 1
GC_HUB_BF16X3 = 0
GC_HUB_F16X2 = 1
GC_HUB_F16 = 2
GC_HUB_F16_MN = 3
GC_HUB_A_BITS = 1 << 6
GC_HUB_TAGGED = 1 << 2
GC_SPMM_B_F16 = 1 << 10


def GC_SPMM_SHRINK(s: int) -> int:  # noqa: N802 - mirrors the C macro
    return (int(s) & 3) << 8


def GC_SPMM_SIG_CHUNKS(c: int) -> int:  # noqa: N802 - mirrors the C macro
    return (int(c) - 1) << 12


def GC_HUB_SIG_CHUNKS(c: int) -> int:  # noqa: N802 - mirrors the C macro
    return (int(c) - 1) << 8


GC_GEMM_TF32 = 1 << 4
GC_GEMM_FP32 = 1 << 5
GC_GEMM_TF32X3 = 1 << 7
GC_SPMM_ROW = 1
GC_SPMM_NNZ_SPLIT = 2
GC_PLAN_LENGTH_CLASSES = 1

GC_OK = 0
GC_ERR_SHAPE = -1
GC_ERR_VALUE = -2
GC_ERR_CUDA = -3
GC_ERR_UNSUPPORTED = -4
GC_ERR_WORKSPACE = -5

HEADER = ROOT / "include" / "gnnc.h"

_lib = None

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_U32 = ctypes.c_uint32
_SZ = ctypes.c_size_t
_F = ctypes.c_float
_i64p = ctypes.POINTER(ctypes.c_int64)

_SIGNATURES = {
    "gc_abi_version": (ctypes.c_int, []),
    "gc_last_error": (ctypes.c_char_p, []),
    "gc_launch_count": (ctypes.c_uint64, []),
    "gc_device_sm_count": (ctypes.c_int, [ctypes.c_int]),
    "gc_spmm_f32": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _I64, _I64, _I64, _I64, _P, _I64, _U32,
                                   ctypes.c_int, _P, _I64, _P, _I64, _P, _SZ, _P]),
    "gc_spmm_gemm_f32": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _I64, _I64, _I64, _I64, _P, _I64,
                                        _P, _I64, _U32, _P]),
    "gc_spmm_plan_count": (ctypes.c_int, [_P, _I64, _I32, _i64p, _i64p, _i64p]),
    "gc_spmm_plan_fill": (ctypes.c_int, [_P, _I64, _I32, _U32, _P, _P]),
    "gc_spmm_default_chunk": (ctypes.c_int32, [_I64, _I64, _I64, ctypes.c_int]),
    "gc_sddmm_f32": (ctypes.c_int, [_P, _P, _P, _P, _I64, _P, _I64, _I64, _I64, _I64, _P, _P]),
    "gc_sddmm_norm_f32": (ctypes.c_int, [_P, _P, _P, _P, _I64, _I64, _P, _P]),
    "gc_gemm_workspace_bytes": (_SZ, [_I64, _I64]),
    "gc_gemm_f16rows_f32": (ctypes.c_int, [_P, _I64, _P, _I64, _I64, _I64, _I64, _P, _P, _I64, _P,
                                           _P, _SZ, _P]),
    "gc_gemm_f32": (ctypes.c_int, [_P, _I64, _P, _I64, _I64, _I64, _I64, _P, _I64, _P, _U32, _P,
                                   _SZ, _P]),
    "gc_scale_rows_f32": (ctypes.c_int, [_P, _P, _I64, _I64, _I64, _P, _I64, _U32, _P]),
    "gc_node_proj_f32": (ctypes.c_int, [_P, _I64, _I64, _I64, _I32, _I64, _P, _P, _P, _P, _P]),
    "gc_gat_sddmm_aggregate_f32": (ctypes.c_int, [_P, _P, _P, _P, _F, _P, _I64, _P, _I64, _P, _I64,
                                                  _I64, _P, _I64,
                                                  _U32, ctypes.c_int, _P, _I64, _P, _I64, _P, _SZ, _P]),
    "gc_gat_aggregate_f32": (ctypes.c_int, [_P, _P, _P, _P, _F, _P, _I64, _P, _I64, _I64, _I64, _P,
                                            _I64,
                                            _U32, ctypes.c_int, _P, _I64, _P, _I64, _P, _SZ, _P]),
    "gc_edge_softmax_heavy_threshold": (ctypes.c_int, [_I64, _I64]),
    "gc_edge_softmax_f32": (ctypes.c_int, [_P, _P, _P, _P, _I32, _F, _I64, _I64, _P, _I64, _P, _P]),
    "gc_attn_sddmm_f32": (ctypes.c_int, [_P, _P, _P, _I64, _P, _I64, _I64, _I32, _P, _P, _F, _I64,
                                         _I64, _P,
                                         _I64, _P, _P, _P]),
    "gc_partition_rows": (ctypes.c_int, [_P, _I64, _I32, _P]),
    "gc_hub_terms_rows": (_I64, [_I64]),
    "gc_hub_pack": (ctypes.c_int, [_P, _I64, _I64, _P, _I64, _P, _I32, _P, _P, _P]),
    "gc_hub_pack_f16rows": (ctypes.c_int, [_P, _I64, _P, _I64, _P, _I64, _P, _I32, _P, _P, _P]),
    "gc_hub_gemm": (ctypes.c_int, [_P, _I64, _I64, _I64, _P, _I64, _I32, _P, _P, _I64, _P, _U32,
                                   _P]),
    "gc_hub_stair_supported": (ctypes.c_int, [_I64]),
    "gc_hub_f16_mn_supported": (ctypes.c_int, [_I64]),
    "gc_zero_rows": (ctypes.c_int, [_P, _I64, _P, _I64, _I64, _P]),
    "gc_hub_stair_pair_bn": (ctypes.c_int, [_I64]),
    "gc_hub_stair_gemm": (ctypes.c_int, [_P, _P, _P, _P, _I32, _P, _P, _P, _I32, _P, _P, _I32, _P,
                                         _I64, _I64, _I32, _P, _P, _I64, _P, _U32, _P]),
    "gc_tag_hub_columns": (ctypes.c_int, [_P, _I64, _P, _P, _P]),
    "gc_pack_rows_f16": (ctypes.c_int, [_P, _I64, _I64, _I64, _P, _P, _I64, _P, _P]),
    "gc_pack_rows_f16_proj": (ctypes.c_int, [_P, _I64, _I64, _I64, _P, _P, _I64, _P, _P, _I32, _P,
                                             _P]),
}


class NativeError(RuntimeError):
    """A kernel entry point returned an error status."""


def header_symbols() -> list[str]:
    """Every function the C ABI header declares."""
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(gc_\w+)\s*\(", text, flags=re.M)))


def load(build_if_missing: bool = True):
    """Load (building first if needed) and bind the kernel library."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB.exists():
        if not build_if_missing:
            raise ImportError(f"{LIB} is missing; run __graft_entry__.build()")
        from ._build import build

        build()
    # GNNC_LIB_PATH: load another build of the same ABI (A/B experiments)
    lib = ctypes.CDLL(os.environ.get("GNNC_LIB_PATH", str(LIB)))
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.gc_abi_version() != ABI_VERSION:
        raise ImportError("libgnnc ABI version mismatch")
    _lib = lib
    return lib


def lib_path() -> Path:
    return LIB


def launch_count() -> int:
    return int(load().gc_launch_count())


def check(rc: int, what: str) -> None:
    """Map a status code to the reference's exception types."""
    if rc == GC_OK:
        return
    msg = (load().gc_last_error() or b"").decode(errors="replace")
    from .sparse import ShapeError  # local import: sparse imports this module

    if rc == GC_ERR_SHAPE:
        raise ShapeError(f"{what}: {msg}")
    if rc == GC_ERR_VALUE:
        raise ValueError(f"{what}: {msg}")
    raise NativeError(f"{what} failed ({rc}): {msg}")
