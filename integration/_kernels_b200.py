"""Drop-in replacement for the reference's native kernel module
``vexsort._kernels`` (pkg/src/vexsort/_kernels.py), binding the B200 C ABI
(include/vexsort_b200.h) with ctypes.

The reference routes every region algorithm to ``_kernels`` whenever
``backend.uses_kernels`` (lanes.py:297): ``from . import _kernels`` at
quicksort.py:124-133, partition.py:49-55 and 134-145, smallsort.py:235-239,
keyvalue.py:90-94, 115-121, 150-161 and 240-249.  Each function below has the
signature of its ``_kernels.py`` twin (same argument order and meaning,
numpy arrays mutated in place, absolute lo/hi, int return values) and calls
the matching ``vx_host_*`` entry point, which copies the region to the B200,
runs the CUDA kernels and copies it back.

Install it in place of the numba module (what a maintainer would do in
vexsort/__init__.py, and what tests/test_gpu_integration.py does):

    import integration._kernels_b200 as kb
    kb.install()          # sys.modules["vexsort._kernels"] = kb

Differences that callers can observe, all allowed by the reference's
contracts: partition LAYOUTS differ (the boundary and the two sides as
multisets are identical), the pivot strategy steers the GPU's sampling but
cannot change a sorted output, and kv order among equal keys is
unspecified (keyvalue.py:230).
"""

from __future__ import annotations

import ctypes
import math
import os
import sys

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.environ.get("VEXSORT_B200_LIB") or os.path.join(os.path.dirname(_HERE), "paper_1704_08579_b200",
                                                         "libvexsort_b200.so")
_L = None
CALLS: dict[str, int] = {}  # per-function call counts (tests prove the routing)


def _lib():
    global _L
    if _L is None:
        L = ctypes.CDLL(_SO)
        i64, i32, u64, vp = ctypes.c_int64, ctypes.c_int, ctypes.c_uint64, ctypes.c_void_p
        L.vx_host_quicksort.argtypes = [i32, vp, i64, i64, i64, i32, i32, i32, u64]
        L.vx_host_kv_quicksort.argtypes = [i32, vp, vp, i64, i64, i64, i32, i32, i32, u64]
        L.vx_host_partition.argtypes = [i32, vp, i64, i64, vp, i64, i32, i32]
        L.vx_host_partition.restype = i64
        L.vx_host_kv_partition.argtypes = [i32, vp, vp, i64, i64, vp, i64, i32, i32]
        L.vx_host_kv_partition.restype = i64
        L.vx_host_smallsort_region.argtypes = [i32, vp, i64, i64]
        L.vx_host_kv_smallsort_region.argtypes = [i32, vp, vp, i64, i64]
        L.vx_host_sort_submit.argtypes = [i32, vp, vp, vp, vp, i64, i64, i64, i32, u64, ctypes.POINTER(ctypes.c_int)]
        L.vx_host_sort_wait.argtypes = [i32]
        L.vx_last_error.restype = ctypes.c_char_p
        L.vx_version.restype = i32
        _L = L
    return _L


def _count(name):
    CALLS[name] = CALLS.get(name, 0) + 1


def _dt(a):
    if a.dtype == np.int32:
        return 0
    if a.dtype == np.float64:
        return 1
    raise TypeError(f"unsupported element dtype {a.dtype}; use int32 or float64")


def _ok(rc):
    if rc < 0:
        raise RuntimeError(_lib().vx_last_error().decode())
    return rc


def _ptr(a):
    assert a.flags.c_contiguous, "regions must be contiguous"
    return ctypes.c_void_p(a.ctypes.data)


def _pivot(a, p):
    """numba compares int32 keys against a float pivot exactly:
    x <= p  <=>  x <= floor(p).  Returns (ctypes pointer, shortcut) where
    shortcut is "none" (no key is <= p) or None."""
    if a.dtype == np.float64:
        return ctypes.byref(ctypes.c_double(float(p))), None
    p = float(p) if not isinstance(p, (int, np.integer)) else int(p)
    if isinstance(p, float):
        if math.isnan(p):
            return None, "none"
        if math.isinf(p):
            return (None, "none") if p < 0 else (ctypes.byref(ctypes.c_int32(2**31 - 1)), None)
        p = math.floor(p)
    if p < -(2**31):
        return None, "none"
    return ctypes.byref(ctypes.c_int32(min(int(p), 2**31 - 1))), None


def available() -> bool:
    try:
        return _lib().vx_version() == 1
    except OSError:
        return False


def quicksort(arr, lane, sort_bound, sentinel, strategy, opt_a, opt_b, seed):  # _kernels.py:378
    _count("quicksort")
    _ok(_lib().vx_host_quicksort(_dt(arr), _ptr(arr), len(arr), int(lane), int(sort_bound), int(strategy),
                                 int(opt_a), int(opt_b), int(seed) & (2**64 - 1)))


def kv_quicksort(keys, vals, lane, sort_bound, sentinel, strategy, opt_a, opt_b, seed):  # _kernels.py:425
    _count("kv_quicksort")
    _ok(_lib().vx_host_kv_quicksort(_dt(keys), _ptr(keys), _ptr(vals), len(keys), int(lane), int(sort_bound),
                                    int(strategy), int(opt_a), int(opt_b), int(seed) & (2**64 - 1)))


def partition(arr, lo, hi, pivot, lane, opt_a, opt_b):  # _kernels.py:257
    _count("partition")
    pc, short = _pivot(arr, pivot)
    if short == "none":
        return int(lo)
    return int(_ok(_lib().vx_host_partition(_dt(arr), _ptr(arr), int(lo), int(hi), pc, int(lane), int(opt_a),
                                            int(opt_b))))


def scalar_partition(arr, lo, hi, pivot):  # _kernels.py:162
    return partition(arr, lo, hi, pivot, 16 if arr.dtype == np.int32 else 8, False, False)


def kv_partition(keys, vals, lo, hi, pivot, lane, opt_a, opt_b):  # _kernels.py:347
    _count("kv_partition")
    pc, short = _pivot(keys, pivot)
    if short == "none":
        return int(lo)
    return int(_ok(_lib().vx_host_kv_partition(_dt(keys), _ptr(keys), _ptr(vals), int(lo), int(hi), pc, int(lane),
                                               int(opt_a), int(opt_b))))


def kv_scalar_partition(keys, vals, lo, hi, pivot):  # _kernels.py:173
    return kv_partition(keys, vals, lo, hi, pivot, 16 if keys.dtype == np.int32 else 8, False, False)


def smallsort_region(arr, lo, length, sentinel):  # _kernels.py:115
    _count("smallsort_region")
    _ok(_lib().vx_host_smallsort_region(_dt(arr), _ptr(arr), int(lo), int(length)))


def kv_smallsort_region(keys, vals, lo, length, sentinel):  # _kernels.py:148
    _count("kv_smallsort_region")
    _ok(_lib().vx_host_kv_smallsort_region(_dt(keys), _ptr(keys), _ptr(vals), int(lo), int(length)))


def quicksort_many(arrays, lane, sort_bound, sentinel, strategy, opt_a, opt_b, seed):
    """``for a in arrays: quicksort(a, ...)`` (quicksort.py:124-133 once per
    array) with the PCIe copies of consecutive arrays overlapped: two sorts
    in flight through vx_host_sort_submit / vx_host_sort_wait."""
    _count("quicksort_many")
    L = _lib()
    pending = []
    for a in arrays:
        if len(pending) == 2:
            _ok(L.vx_host_sort_wait(pending.pop(0)))
        t = ctypes.c_int(-1)
        _ok(L.vx_host_sort_submit(_dt(a), _ptr(a), None, _ptr(a), None, len(a), lane, sort_bound, strategy,
                                  seed & (2**64 - 1), ctypes.byref(t)))
        pending.append(t.value)
    for t in pending:
        _ok(L.vx_host_sort_wait(t))


def install() -> None:
    """Route the reference's ``from . import _kernels`` to this module."""
    sys.modules["vexsort._kernels"] = sys.modules[__name__]
    pkg = sys.modules.get("vexsort")
    if pkg is not None:
        pkg._kernels = sys.modules[__name__]
