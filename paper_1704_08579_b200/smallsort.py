"""Small-region bitonic sort API (mirror of vexsort/smallsort.py) plus the
batched CSR entry point of config 2.

``sort_small_region(region)`` keeps the reference contract: n <= 16*lanes
(256 int32 / 128 float64, AssertionError beyond, smallsort.py:218-252),
sentinel padding by count.  ``sort_segments(values, offsets)`` sorts every
CSR segment (length <= 256 for both kinds) with one warp-register bitonic
network per segment in a single launch (csrc/bitonic.cuh).
"""

from __future__ import annotations

from ._lib import check, lib
from ._region import check_region, dev_ptr, host_ptr, on_device, stream_of, workspace
from .lanes import ElemKind, get_backend, is_device
from .quicksort import MAX_PACKS, SortConfig, sort_with_config

__all__ = ["MAX_PACKS", "MAX_SEGMENT", "max_small_length", "sort_small_region", "sort_segments"]

MAX_SEGMENT = 256


def max_small_length(kind: ElemKind) -> int:
    return MAX_PACKS * kind.lanes


def sort_small_region(region, backend=None) -> None:
    """Sort a region of length <= 16*L in place."""
    n = len(region)
    if n < 2:
        return
    kind = check_region(region)
    if backend is None:
        backend = get_backend("auto", kind)
    assert n <= MAX_PACKS * backend.lanes, "region exceeds small-sort capacity"
    if is_device(region):
        sort_with_config(region, SortConfig(sort_bound=MAX_PACKS * backend.lanes))
        return
    check(lib().vx_host_smallsort_region(kind.code, host_ptr(region), 0, n), "sort_small_region")


def sort_segments(values, offsets, payload=None, *, validate: bool = True) -> None:
    """Sort each CSR segment values[offsets[s]:offsets[s+1]] ascending in
    place (device tensors; offsets int64 of length nseg+1).  With `payload`
    (same length and element width), pairs move together and are swapped only
    on strict key inversion, as in the reference's kv network.  validate=True
    synchronises and raises AssertionError if a segment exceeds 256 or an
    offset lies outside [0, len(values)] (such segments are never touched)."""
    import torch

    kind = check_region(values)
    assert is_device(values), "sort_segments takes CUDA tensors"
    assert offsets.dtype == torch.int64 and offsets.ndim == 1 and offsets.is_contiguous()
    assert offsets.device == values.device
    if payload is not None:
        assert payload.is_cuda and len(payload) == len(values)
        assert payload.element_size() == values.element_size() and payload.is_contiguous()
    nseg = len(offsets) - 1
    if nseg <= 0:
        return
    L = lib()
    with on_device(values):
        ws = workspace(256, values.device)
        st = stream_of(values)
        check(L.vx_sort_segments(kind.code, dev_ptr(values), dev_ptr(payload) if payload is not None else None,
                                 len(values), dev_ptr(offsets), nseg, dev_ptr(ws), ws.numel(), st), "sort_segments")
        if validate:
            check(L.vx_segments_status(dev_ptr(ws), st), "sort_segments")
