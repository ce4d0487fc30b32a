"""ctypes binding of libvexsort_b200.so (the C ABI in include/vexsort_b200.h).

There is no CPU fallback: if the shared library or a CUDA device is missing,
every entry point raises :class:`BackendUnavailable` (the reference's
fail-fast contract for an unavailable native backend, lanes.py:448-457).
ctypes releases the GIL for the duration of each call.
"""

from __future__ import annotations

import ctypes
import os
import threading

__all__ = ["BackendUnavailable", "lib", "check", "lib_path", "VX_I32", "VX_F64", "SortConfigC", "SortStatsC"]

VX_I32, VX_F64 = 0, 1
VX_SORT_GRAPH, VX_SORT_EAGER = 1, 2  # vx_sort_config.flags
_HERE = os.path.dirname(os.path.abspath(__file__))
# VEXSORT_B200_LIB overrides the library path (tuning experiments only)
_SO = os.environ.get("VEXSORT_B200_LIB") or os.path.join(_HERE, "libvexsort_b200.so")


class BackendUnavailable(RuntimeError):
    """The B200 backend cannot run here (library not built or no GPU)."""


class SortConfigC(ctypes.Structure):
    _fields_ = [
        ("sort_bound", ctypes.c_int64),
        ("pivot_strategy", ctypes.c_int32),
        ("skip_empty_stores", ctypes.c_int32),
        ("swap_buffered", ctypes.c_int32),
        ("flags", ctypes.c_int32),
        ("pivot_seed", ctypes.c_uint64),
    ]


class SortStatsC(ctypes.Structure):
    _fields_ = [
        ("err", ctypes.c_uint32),
        ("levels", ctypes.c_uint32),
        ("launches", ctypes.c_uint32),
        ("reserved", ctypes.c_uint32),
        ("scatter_elems", ctypes.c_uint64),
        ("finish_elems", ctypes.c_uint64),
        ("local_elems", ctypes.c_uint64),
    ]


_lock = threading.Lock()
_lib = None


def lib_path() -> str:
    return _SO


def _declare(L):
    i64, i32, u64, vp, sz = ctypes.c_int64, ctypes.c_int, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_size_t
    sigs = {
        "vx_last_error": ([], ctypes.c_char_p),
        "vx_version": ([], i32),
        "vx_sort_workspace_bytes": ([i32, i32, i64], sz),
        "vx_sort": ([i32, vp, vp, i64, ctypes.POINTER(SortConfigC), vp, sz, vp], i32),
        "vx_sort_into": ([i32, vp, vp, vp, vp, i64, ctypes.POINTER(SortConfigC), vp, sz, vp], i32),
        "vx_profile_enable": ([i32], i32),
        "vx_profile_reset": ([], i32),
        "vx_profile_read": ([ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_double),
                             ctypes.POINTER(ctypes.c_uint64), i32], i32),
        "vx_partition_workspace_bytes": ([i32, i64], sz),
        "vx_partition": ([i32, vp, vp, vp, vp, i64, vp, vp, vp, sz, vp], i32),
        "vx_sort_segments": ([i32, vp, vp, i64, vp, i64, vp, sz, vp], i32),
        "vx_sort_status": ([vp, i64, vp, ctypes.POINTER(SortStatsC)], i32),
        "vx_segments_status": ([vp, vp], i32),
        "vx_bucket_partition_workspace_bytes": ([i32, i32], sz),
        "vx_bucket_partition": ([i32, vp, vp, i64, u64, vp, vp, i32, vp, vp, sz, vp], i32),
        "vx_select_splitters": ([i32, vp, vp, i64, i32, vp, vp, vp], i32),
        "vx_bucket_counts": ([i32, vp, i64, u64, vp, vp, i32, vp, vp], i32),
        "vx_bucket_scatter_to": ([i32, vp, i64, u64, vp, vp, i32, vp, vp, vp, sz, vp], i32),
        "vx_ipc_alloc": ([sz, ctypes.POINTER(ctypes.c_void_p)], i32),
        "vx_ipc_free": ([vp], i32),
        "vx_ipc_handle": ([vp, vp], i32),
        "vx_ipc_open": ([vp, ctypes.POINTER(ctypes.c_void_p)], i32),
        "vx_ipc_close": ([vp], i32),
        "vx_sort_from_ptr": ([i32, u64, vp, i64, ctypes.POINTER(SortConfigC), vp, sz, vp], i32),
        "vx_generate": ([i32, i32, vp, i64, u64, u64, i64, vp], i32),
        "vx_verify": ([i32, vp, vp, i64, i32, vp, i64, vp, vp], i32),
        "vx_host_quicksort": ([i32, vp, i64, i64, i64, i32, i32, i32, u64], i32),
        "vx_host_kv_quicksort": ([i32, vp, vp, i64, i64, i64, i32, i32, i32, u64], i32),
        "vx_host_partition": ([i32, vp, i64, i64, vp, i64, i32, i32], i64),
        "vx_host_kv_partition": ([i32, vp, vp, i64, i64, vp, i64, i32, i32], i64),
        "vx_host_scalar_partition": ([i32, vp, i64, i64, vp], i64),
        "vx_host_kv_scalar_partition": ([i32, vp, vp, i64, i64, vp], i64),
        "vx_host_smallsort_region": ([i32, vp, i64, i64], i32),
        "vx_host_kv_smallsort_region": ([i32, vp, vp, i64, i64], i32),
        "vx_host_sort_submit": ([i32, vp, vp, vp, vp, i64, i64, i64, i32, u64, ctypes.POINTER(ctypes.c_int)], i32),
        "vx_host_sort_wait": ([i32], i32),
        "vx_host_pin": ([vp, sz], i32),
        "vx_host_unpin": ([vp], i32),
        "vx_host_release": ([], i32),
    }
    for name, (args, res) in sigs.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res


def lib() -> ctypes.CDLL:
    """Load (once) and return the C-ABI library; raise if unusable."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(_SO):
                raise BackendUnavailable(
                    f"B200 kernels not built ({_SO} missing); run __graft_entry__.build()")
            try:
                L = ctypes.CDLL(_SO)
            except OSError as exc:  # pragma: no cover - depends on the host
                raise BackendUnavailable(f"cannot load {_SO}: {exc}") from exc
            _declare(L)
            _lib = L
    return _lib


class VexsortError(RuntimeError):
    pass


def check(rc: int, what: str = "") -> int:
    """Map C-ABI status codes onto the reference's exception types."""
    if rc >= 0:
        return rc
    msg = (lib().vx_last_error() or b"").decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == -2:
        raise TypeError(text)
    if rc in (-1, -6):
        raise AssertionError(text)  # reference contract violations are asserts
    raise VexsortError(text)
