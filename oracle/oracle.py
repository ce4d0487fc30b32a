"""ctypes + numpy front end of the CPU oracle (test infrastructure only).

Function names and argument meanings follow the reference's native kernel
module ``pkg/src/vexsort/_kernels.py`` (cited per function) so the parity
tests read like the reference's own tests.  Arrays are numpy, mutated in
place, exactly as the reference does.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

__all__ = [
    "lib",
    "build",
    "I32_SENTINEL",
    "F64_SENTINEL",
    "lanes_for",
    "sentinel_for",
    "default_bound",
    "smallsort_region",
    "kv_smallsort_region",
    "scalar_partition",
    "kv_scalar_partition",
    "partition",
    "kv_partition",
    "quicksort",
    "kv_quicksort",
    "sort",
    "kv_sort",
    "partition_region",
    "kv_partition_region",
    "median3_index",
    "oracle_sort",
    "oracle_partition",
    "oracle_kv_sort",
    "max_threads",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")

# lanes.py:60-61 -- lane count and padding sentinel per element kind
I32_SENTINEL = 2**31 - 1
F64_SENTINEL = math.inf
_STRATEGIES = ("median3", "middle", "random")  # quicksort.py:20


def build(force: bool = False) -> str:
    """Compile liboracle.so with the committed Makefile."""
    if force or not os.path.exists(_SO) or (
        os.path.getmtime(_SO) < os.path.getmtime(os.path.join(_HERE, "vexsort_oracle.c"))
    ):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        i64, i32, u64, vp, f64 = (ctypes.c_int64, ctypes.c_int, ctypes.c_uint64,
                                  ctypes.c_void_p, ctypes.c_double)
        k32 = ctypes.c_int32
        for suf, kt in (("i32", k32), ("f64", f64)):
            getattr(L, f"vxo_smallsort_region_{suf}").argtypes = [vp, i64, i64, kt]
            getattr(L, f"vxo_smallsort_region_{suf}").restype = i32
            getattr(L, f"vxo_scalar_partition_{suf}").argtypes = [vp, i64, i64, kt]
            getattr(L, f"vxo_scalar_partition_{suf}").restype = i64
            getattr(L, f"vxo_partition_{suf}").argtypes = [vp, i64, i64, kt, i64, i32, i32]
            getattr(L, f"vxo_partition_{suf}").restype = i64
            getattr(L, f"vxo_quicksort_{suf}").argtypes = [vp, i64, i64, i64, kt, i32, i32, i32, u64]
            getattr(L, f"vxo_quicksort_{suf}").restype = i32
            getattr(L, f"vxo_quicksort_mt_{suf}").argtypes = [vp, i64, i64, i64, kt, i32, i32, i32, u64, i32]
            getattr(L, f"vxo_quicksort_mt_{suf}").restype = i32
        for suf, kt in (("kvi32", k32), ("kvf64", f64)):
            getattr(L, f"vxo_kv_smallsort_region_{suf}").argtypes = [vp, vp, i64, i64, kt]
            getattr(L, f"vxo_kv_smallsort_region_{suf}").restype = i32
            getattr(L, f"vxo_kv_scalar_partition_{suf}").argtypes = [vp, vp, i64, i64, kt]
            getattr(L, f"vxo_kv_scalar_partition_{suf}").restype = i64
            getattr(L, f"vxo_kv_partition_{suf}").argtypes = [vp, vp, i64, i64, kt, i64, i32, i32]
            getattr(L, f"vxo_kv_partition_{suf}").restype = i64
            getattr(L, f"vxo_kv_quicksort_{suf}").argtypes = [vp, vp, i64, i64, i64, kt, i32, i32, i32, u64, i32]
            getattr(L, f"vxo_kv_quicksort_{suf}").restype = i32
        L.vxo_max_threads.restype = i32
        _lib = L
    return _lib


def max_threads() -> int:
    return int(lib().vxo_max_threads())


def _suffix(arr) -> str:
    if arr.dtype == np.int32:
        return "i32"
    if arr.dtype == np.float64:
        return "f64"
    raise TypeError(f"unsupported element dtype {arr.dtype}; use int32 or float64")


def _check(arr):
    assert isinstance(arr, np.ndarray) and arr.ndim == 1 and arr.flags.c_contiguous
    return arr.ctypes.data


def lanes_for(arr) -> int:
    return 16 if _suffix(arr) == "i32" else 8  # 512-bit packs, lanes.py:60-61


def sentinel_for(arr):
    return I32_SENTINEL if _suffix(arr) == "i32" else F64_SENTINEL


def default_bound(arr) -> int:
    return 16 * lanes_for(arr)  # quicksort.py:49-52, MAX_PACKS * lanes


def _pivot_c(arr, pivot):
    """Pivot as the C kernel's key type.  For int32 regions a non-integral
    pivot p compares like floor(p) (numba compares mathematically)."""
    if arr.dtype == np.int32:
        p = math.floor(pivot)
        return int(min(max(p, -(2**31) - 1), 2**31 - 1)) if p >= -(2**31) else None
    return float(pivot)


# -- _kernels.py signatures ----------------------------------------------------


def smallsort_region(arr, lo, length, sentinel):
    """_kernels.smallsort_region (_kernels.py:115-126)."""
    rc = getattr(lib(), f"vxo_smallsort_region_{_suffix(arr)}")(_check(arr), lo, length, sentinel)
    assert rc == 0


def kv_smallsort_region(keys, vals, lo, length, sentinel):
    """_kernels.kv_smallsort_region (_kernels.py:148-160)."""
    _check_kv(keys, vals)
    rc = getattr(lib(), f"vxo_kv_smallsort_region_kv{_suffix(keys)}")(
        _check(keys), _check(vals), lo, length, sentinel)
    assert rc == 0


def scalar_partition(arr, lo, hi, pivot) -> int:
    """_kernels.scalar_partition (_kernels.py:162-171)."""
    p = _pivot_c(arr, pivot)
    if p is None:  # pivot below every int32: nothing is low
        return lo
    return int(getattr(lib(), f"vxo_scalar_partition_{_suffix(arr)}")(_check(arr), lo, hi, p))


def kv_scalar_partition(keys, vals, lo, hi, pivot) -> int:
    """_kernels.kv_scalar_partition (_kernels.py:173-185)."""
    _check_kv(keys, vals)
    p = _pivot_c(keys, pivot)
    if p is None:
        return lo
    return int(getattr(lib(), f"vxo_kv_scalar_partition_kv{_suffix(keys)}")(
        _check(keys), _check(vals), lo, hi, p))


def partition(arr, lo, hi, pivot, lane, opt_a=False, opt_b=False) -> int:
    """_kernels.partition (_kernels.py:257-262)."""
    p = _pivot_c(arr, pivot)
    if p is None:
        return lo
    r = int(getattr(lib(), f"vxo_partition_{_suffix(arr)}")(
        _check(arr), lo, hi, p, lane, int(opt_a), int(opt_b)))
    assert r >= 0
    return r


def kv_partition(keys, vals, lo, hi, pivot, lane, opt_a=False, opt_b=False) -> int:
    """_kernels.kv_partition (_kernels.py:347-356)."""
    _check_kv(keys, vals)
    p = _pivot_c(keys, pivot)
    if p is None:
        return lo
    r = int(getattr(lib(), f"vxo_kv_partition_kv{_suffix(keys)}")(
        _check(keys), _check(vals), lo, hi, p, lane, int(opt_a), int(opt_b)))
    assert r >= 0
    return r


def quicksort(arr, lane, sort_bound, sentinel, strategy=0, opt_a=False, opt_b=False,
              seed=0, nthreads=1):
    """_kernels.quicksort (_kernels.py:378-423).  nthreads != 1 runs the
    OpenMP task-parallel variant (identical output)."""
    suf = _suffix(arr)
    seed = int(seed) & (2**64 - 1)
    if nthreads == 1:
        rc = getattr(lib(), f"vxo_quicksort_{suf}")(
            _check(arr), len(arr), lane, sort_bound, sentinel, strategy,
            int(opt_a), int(opt_b), seed)
    else:
        rc = getattr(lib(), f"vxo_quicksort_mt_{suf}")(
            _check(arr), len(arr), lane, sort_bound, sentinel, strategy,
            int(opt_a), int(opt_b), seed, nthreads)
    assert rc == 0


def kv_quicksort(keys, vals, lane, sort_bound, sentinel, strategy=0, opt_a=False,
                 opt_b=False, seed=0, nthreads=1):
    """_kernels.kv_quicksort (_kernels.py:425-482)."""
    _check_kv(keys, vals)
    rc = getattr(lib(), f"vxo_kv_quicksort_kv{_suffix(keys)}")(
        _check(keys), _check(vals), len(keys), lane, sort_bound, sentinel, strategy,
        int(opt_a), int(opt_b), int(seed) & (2**64 - 1), nthreads)
    assert rc == 0


def _check_kv(keys, vals):
    # keyvalue.py:44-47
    assert len(keys) == len(vals), "keys and values must have equal length"
    assert keys.dtype.itemsize == vals.dtype.itemsize, \
        "values must have the same element width as keys"


# -- public-API restatements (quicksort.py / partition.py / keyvalue.py) -------


def sort(arr, sort_bound=None, pivot_strategy="median3", seed=0, nthreads=1):
    """vexsort.sort / sort_with_config on the native backend
    (quicksort.py:115-143)."""
    if len(arr) < 2:
        return
    bound = default_bound(arr) if sort_bound is None else sort_bound
    quicksort(arr, lanes_for(arr), bound, sentinel_for(arr),
              _STRATEGIES.index(pivot_strategy), seed=seed, nthreads=nthreads)


def kv_sort(keys, vals, sort_bound=None, pivot_strategy="median3", seed=0, nthreads=1):
    """vexsort.kv_sort (keyvalue.py:228-252)."""
    _check_kv(keys, vals)
    if len(keys) < 2:
        return
    bound = default_bound(keys) if sort_bound is None else sort_bound
    kv_quicksort(keys, vals, lanes_for(keys), bound, sentinel_for(keys),
                 _STRATEGIES.index(pivot_strategy), seed=seed, nthreads=nthreads)


def partition_region(arr, pivot, opt_a=False, opt_b=False) -> int:
    """vexsort.partition_region (partition.py:115-145): n <= 2L uses the
    scalar partition, else the two-cursor vector partition."""
    n = len(arr)
    L = lanes_for(arr)
    if n <= 2 * L:
        return scalar_partition(arr, 0, n, pivot)
    return partition(arr, 0, n, pivot, L, opt_a, opt_b)


def kv_partition_region(keys, vals, pivot, opt_a=False, opt_b=False) -> int:
    """vexsort.kv_partition_region (keyvalue.py:138-161)."""
    _check_kv(keys, vals)
    n = len(keys)
    L = lanes_for(keys)
    if n <= 2 * L:
        return kv_scalar_partition(keys, vals, 0, n, pivot)
    return kv_partition(keys, vals, 0, n, pivot, L, opt_a, opt_b)


def median3_index(arr, lo, hi) -> int:
    """select_pivot(..., "median3") (quicksort.py:55-74) over [lo, hi]."""
    mid = (lo + hi) // 2
    a, b, c = arr[lo], arr[mid], arr[hi]
    if b <= a <= c or c <= a <= b:
        return lo
    if a <= b <= c or c <= b <= a:
        return mid
    return hi


# -- oracle.py restatements -----------------------------------------------------


def oracle_sort(region) -> None:
    """oracle.py:15-21 -- the platform sort."""
    region[:] = np.sort(region)


def oracle_partition(region, pivot) -> int:
    """oracle.py:35-45 -- stable two-sided partition; returns count(<= pivot)."""
    arr = np.asarray(region)
    mask = arr <= pivot
    low, high = arr[mask], arr[~mask]
    region[:len(low)] = low
    region[len(low):] = high
    return len(low)


def oracle_kv_sort(keys, values) -> None:
    """oracle.py:48-54 -- stable by original index."""
    order = np.argsort(keys, kind="stable")
    keys[:] = keys[order]
    values[:] = values[order]
