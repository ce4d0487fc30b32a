"""Pivot partition API (mirror of vexsort/partition.py).

``partition_region(region, pivot)`` partitions in place and returns the
boundary: region[:b] <= pivot < region[b:], b = count(<= pivot)
(partition.py:115-175).  On the device it runs the single-pass
decoupled-look-back kernel (csrc/partition2.cuh) out of place; pass
``out=`` to keep the result there (one read + one write of the data, the
config-3 roofline), otherwise the result is copied back into ``region``.
"""

from __future__ import annotations

import ctypes

from ._lib import check, lib
from ._region import check_region, dev_ptr, host_ptr, on_device, pivot_for, stream_of, workspace
from .lanes import get_backend, is_device

__all__ = ["partition_region", "scalar_partition"]


def _device_partition(kind, keys, values, pivot_c, out_keys, out_values):
    import torch

    n = len(keys)
    L = lib()
    with on_device(keys):
        ws = workspace(L.vx_partition_workspace_bytes(kind.code, n), keys.device)
        split = torch.empty(1, dtype=torch.int64, device=keys.device)
        check(L.vx_partition(kind.code, dev_ptr(keys), dev_ptr(values) if values is not None else None,
                             dev_ptr(out_keys), dev_ptr(out_values) if out_values is not None else None, n,
                             ctypes.byref(pivot_c), dev_ptr(split), dev_ptr(ws), ws.numel(), stream_of(keys)),
              "partition")
    return split


def partition_region(region, pivot, backend=None, *, skip_empty_stores: bool = False,
                     swap_buffered: bool = False, out=None) -> int:
    """Partition `region` around `pivot`; return the boundary (count of
    elements <= pivot).  The multiset is preserved.  The two flags are the
    reference's CPU store-pattern variants and are accepted as no-ops."""
    kind = check_region(region)
    if backend is None:
        backend = get_backend("auto", kind)
    n = len(region)
    pc, short = pivot_for(kind, pivot)
    if short is not None:
        if out is not None:
            out.copy_(region)
        return 0 if short == "none" else n
    if n == 0:
        return 0
    if is_device(region):
        import torch

        dst = out if out is not None else torch.empty_like(region)
        assert dst.is_cuda and dst.dtype == region.dtype and len(dst) == n and dst.is_contiguous()
        split = _device_partition(kind, region, None, pc, dst, None)
        if out is None:
            region.copy_(dst)
        return int(split.item())
    assert out is None, "out= is a device-path option"
    L = lib()
    return int(check(L.vx_host_partition(kind.code, host_ptr(region), 0, n, ctypes.byref(pc), backend.lanes,
                                         int(skip_empty_stores), int(swap_buffered)), "partition"))


def scalar_partition(region, pivot) -> int:
    """The reference's scalar twin (partition.py:44-66): same boundary."""
    return partition_region(region, pivot)
