"""ctypes binding of libbbx.so (include/bbx.h).

The product has no CPU fallback: if the library cannot be loaded, every
device entry point raises.  The library is built in-tree by
``paper_2306_12517_b200._build.build()`` (called from __graft_entry__.build()).
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from . import errors as E

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "libbbx.so"

c_i32, c_i64, c_u64, c_vp, c_dbl, c_flt = (ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p,
                                           ctypes.c_double, ctypes.c_float)


class BbxOp(ctypes.Structure):
    _fields_ = [("kind", c_i32), ("h", c_i32), ("w", c_i32), ("dtype", c_i32), ("p", c_dbl),
                ("scale", c_dbl * 2), ("ratio", c_dbl * 2), ("mean", c_flt * 4), ("std", c_flt * 4)]


class FieldInfo(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 64), ("kind", c_i32), ("array_dtype", c_i32), ("ndims", c_i32),
                ("dims", c_i64 * 4), ("max_height", c_i32), ("max_width", c_i32), ("channels", c_i32),
                ("cell_offset", c_i32)]


class HeaderInfo(ctypes.Structure):
    _fields_ = [("num_samples", c_i64), ("page_size", c_i64), ("data_table_offset", c_i64),
                ("heap_offset", c_i64), ("alloc_table_offset", c_i64), ("num_fields", c_i32),
                ("row_width", c_i32)]


class LoaderStats(ctypes.Structure):
    _fields_ = [("batches", c_i64), ("samples", c_i64), ("h2d_bytes", c_i64), ("d2h_bytes", c_i64),
                ("kernel_launches", c_i64), ("stage_seconds", c_dbl), ("wait_seconds", c_dbl),
                ("kernel_seconds", c_dbl), ("kernel_timed", c_i64), ("kernel_bytes", c_i64),
                ("zero_copy_bytes", c_i64), ("gap_seconds", c_dbl), ("h2d_late_seconds", c_dbl),
                ("timed_batches", c_i64), ("page_fetches", c_i64), ("page_reloads", c_i64),
                ("io_reads", c_i64), ("numa_node", c_i64), ("staging_threads", c_i64), ("staging_cpus", c_i64),
                ("pipeline_seconds", c_dbl)]


# bbx_status -> exception class (errors.py:4-57)
STATUS_EXC = {
    1: E.InvalidFile, 2: E.BadMagic, 3: E.UnsupportedVersion, 4: E.SchemaMismatch, 5: E.SpecMismatch,
    6: E.CorruptPayload, 7: E.IndexOutOfRange, 8: E.CapacityTooSmall, 9: E.ShutdownError, 10: E.DeviceError,
    11: E.InvalidHeader, 12: ValueError,
}

# op kinds (bbx_op_kind) and dtypes (bbx_dtype)
OP_DECODE, OP_ARRAYREAD, OP_TOFLOAT, OP_NORMALIZE, OP_FLIP, OP_CROP, OP_RESIZE, OP_RRC, OP_CENTERCROP, \
    OP_NORMALIZE_PC, OP_CAST = range(11)
DT_U8, DT_I64, DT_F32, DT_F64, DT_F16, DT_BF16 = range(6)

_lib = None


def lib():
    """Load libbbx.so (building it first when the sources are newer)."""
    global _lib
    if _lib is not None:
        return _lib
    if os.environ.get("BBX_NO_BUILD") != "1":
        from . import _build
        try:
            _build.build()
        except Exception as e:  # pragma: no cover - surfaced below if the .so is missing too
            if not LIB_PATH.exists():
                raise E.DeviceError(f"libbbx.so is missing and could not be built: {e}") from e
    if not LIB_PATH.exists():
        raise E.DeviceError(f"libbbx.so not found at {LIB_PATH}; run __graft_entry__.build()")
    return _bind(ctypes.CDLL(str(LIB_PATH)))


def _bind(L):
    global _lib
    P = ctypes.POINTER
    sig = {
        "bbx_last_error": (ctypes.c_char_p, []),
        "bbx_version": (ctypes.c_char_p, []),
        "bbx_dataset_open": (c_i32, [ctypes.c_char_p, P(c_vp)]),
        "bbx_dataset_close": (None, [c_vp]),
        "bbx_dataset_header": (c_i32, [c_vp, P(HeaderInfo)]),
        "bbx_dataset_field": (c_i32, [c_vp, ctypes.c_int, P(FieldInfo)]),
        "bbx_dataset_row": (c_i32, [c_vp, c_i64, c_vp, c_i32]),
        "bbx_dataset_make_resident": (c_i32, [c_vp, ctypes.c_int]),
        "bbx_dataset_page_map": (c_i32, [c_vp, c_vp]),
        "bbx_dataset_pin_host": (c_i32, [c_vp, ctypes.c_int]),
        "bbx_epoch_order": (c_i32, [ctypes.c_int, c_u64, c_u64, c_i64, c_vp, c_i64, c_vp]),
        "bbx_loader_create": (c_i32, [c_vp, ctypes.c_int, c_i32, c_i32, c_i32, P(c_vp)]),
        "bbx_loader_destroy": (None, [c_vp]),
        "bbx_loader_add_field": (c_i32, [c_vp, c_i32, P(BbxOp), c_i32, P(c_i32), P(c_i64), P(c_i32), P(c_i32)]),
        "bbx_loader_add_scalar": (c_i32, [c_vp, c_i32, P(c_i32)]),
        "bbx_loader_bind": (c_i32, [c_vp, c_i32, c_i32, c_vp]),
        "bbx_loader_submit": (c_i32, [c_vp, c_i32, c_vp, c_i32, c_u64, c_u64]),
        "bbx_loader_wait": (c_i32, [c_vp, c_i32, P(c_i64)]),
        "bbx_loader_stream_wait": (c_i32, [c_vp, c_i32, c_vp]),
        "bbx_loader_release": (c_i32, [c_vp, c_i32, c_vp]),
        "bbx_loader_step": (c_i32, [c_vp, c_i32, c_i32, c_vp, c_i32, c_u64, c_u64, c_i32, c_vp, P(c_i64)]),
        "bbx_loader_drain": (c_i32, [c_vp]),
        "bbx_loader_get_stats": (c_i32, [c_vp, P(LoaderStats)]),
        "bbx_loader_reset_stats": (c_i32, [c_vp]),
        "bbx_loader_compute_stream": (c_vp, [c_vp]),
        "bbx_loader_set_profiling": (c_i32, [c_vp, ctypes.c_int]),
        "bbx_loader_set_zero_copy": (c_i32, [c_vp, ctypes.c_int]),
        "bbx_loader_set_option": (c_i32, [c_vp, ctypes.c_char_p, c_i64]),
        "bbx_loader_prefetch_headers": (c_i32, [c_vp, c_vp, c_i64]),
        "bbx_decode_image": (c_i32, [c_i32, c_i32, c_i32, c_i32, c_vp, c_i64, c_vp, ctypes.c_int]),
        "bbx_jpeg_check": (c_i32, [c_i32, c_i32, c_i32, c_vp, c_i64]),
        "bbx_loader_set_page_pool": (c_i32, [c_vp, c_i64, c_dbl]),
        "bbx_loader_plan_epoch": (c_i32, [c_vp, c_vp, c_vp, c_i32, P(c_i64), P(c_i64)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


EXPORTED = ("bbx_last_error", "bbx_version", "bbx_dataset_open", "bbx_dataset_close", "bbx_dataset_header",
            "bbx_dataset_field", "bbx_dataset_row", "bbx_dataset_make_resident", "bbx_dataset_pin_host",
            "bbx_dataset_page_map",
            "bbx_epoch_order", "bbx_loader_create", "bbx_loader_destroy", "bbx_loader_add_field",
            "bbx_loader_add_scalar", "bbx_loader_bind", "bbx_loader_submit", "bbx_loader_wait",
            "bbx_loader_stream_wait", "bbx_loader_release", "bbx_loader_step", "bbx_loader_drain", "bbx_loader_get_stats",
            "bbx_loader_reset_stats", "bbx_loader_compute_stream", "bbx_loader_set_profiling",
            "bbx_loader_set_zero_copy", "bbx_loader_set_option", "bbx_loader_prefetch_headers",
            "bbx_decode_image", "bbx_jpeg_check", "bbx_loader_set_page_pool", "bbx_loader_plan_epoch")


def last_error() -> str:
    return lib().bbx_last_error().decode(errors="replace")


def check(status: int, prefix: str = "") -> None:
    if status == 0:
        return
    exc = STATUS_EXC.get(status, E.BboxError)
    msg = last_error()
    raise exc(prefix + msg if prefix else msg)
