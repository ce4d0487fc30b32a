"""Key/value API (mirror of vexsort/keyvalue.py).

Keys and values are twin 1-D arrays of equal length and equal element width
(keyvalue.py:44-47); values are moved as raw bits.  ``kv_sort`` sorts by key
(value order among equal keys unspecified, keyvalue.py:228-252);
``sort_kv`` is the north-star spelling of the same entry point.
"""

from __future__ import annotations

import ctypes

from ._lib import check, lib
from ._region import check_kv, dev_ptr, host_ptr, pivot_for, stream_of, workspace
from .lanes import get_backend, is_device
from .partition import _device_partition
from .quicksort import MAX_PACKS, SortConfig, _PIVOT_STRATEGIES, _U64, _device_sort, _resolve_bound

__all__ = ["kv_sort", "sort_kv", "kv_partition_region", "kv_sort_small_region", "kv_scalar_partition"]


def kv_sort(keys, values, config: SortConfig | None = None) -> None:
    """Sort keys ascending in place, carrying values along."""
    kind = check_kv(keys, values)
    config = config or SortConfig()
    n = len(keys)
    if n < 2:
        return
    backend = get_backend(config.backend, kind)
    bound = _resolve_bound(config, backend.lanes)
    L = lib()
    if is_device(keys):
        _device_sort(kind, keys, values, keys, values, config, bound, True, "kv_sort")
        return
    check(L.vx_host_kv_quicksort(kind.code, host_ptr(keys), host_ptr(values), n, backend.lanes, bound,
                                 _PIVOT_STRATEGIES.index(config.pivot_strategy), int(config.skip_empty_stores),
                                 int(config.swap_buffered), int(config.pivot_seed) & _U64), "kv_sort")


sort_kv = kv_sort


def kv_partition_region(keys, values, pivot, backend=None, *, skip_empty_stores: bool = False,
                        swap_buffered: bool = False, out=None) -> int:
    """Partition keys around `pivot`, moving values with the same moves;
    return the boundary (keyvalue.py:138-225).  out=(keys_out, values_out)
    keeps the device result out of place."""
    kind = check_kv(keys, values)
    if backend is None:
        backend = get_backend("auto", kind)
    n = len(keys)
    pc, short = pivot_for(kind, pivot)
    if short is not None:
        if out is not None:
            out[0].copy_(keys)
            out[1].copy_(values)
        return 0 if short == "none" else n
    if n == 0:
        return 0
    if is_device(keys):
        import torch

        if out is not None:
            ok, ov = out
        else:
            ok, ov = torch.empty_like(keys), torch.empty_like(values)
        split = _device_partition(kind, keys, values, pc, ok, ov)
        if out is None:
            keys.copy_(ok)
            values.copy_(ov)
        return int(split.item())
    assert out is None, "out= is a device-path option"
    return int(check(lib().vx_host_kv_partition(kind.code, host_ptr(keys), host_ptr(values), 0, n,
                                                ctypes.byref(pc), backend.lanes, int(skip_empty_stores),
                                                int(swap_buffered)), "kv_partition_region"))


def kv_scalar_partition(keys, values, pivot) -> int:
    return kv_partition_region(keys, values, pivot)


def kv_sort_small_region(keys, values, backend=None) -> None:
    """Sort a (keys, values) pair of length <= 16*L in place by key."""
    kind = check_kv(keys, values)
    if backend is None:
        backend = get_backend("auto", kind)
    n = len(keys)
    if n < 2:
        return
    assert n <= MAX_PACKS * backend.lanes, "region exceeds small-sort capacity"
    if is_device(keys):
        kv_sort(keys, values, SortConfig(sort_bound=MAX_PACKS * backend.lanes))
        return
    check(lib().vx_host_kv_smallsort_region(kind.code, host_ptr(keys), host_ptr(values), 0, n),
          "kv_sort_small_region")
