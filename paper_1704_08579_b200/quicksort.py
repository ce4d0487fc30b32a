"""Hybrid quicksort API (mirror of vexsort/quicksort.py).

``sort`` / ``sort_with_config`` keep the reference's names, config object,
validation and in-place semantics (quicksort.py:28-52, 115-143).  The work
runs in the device-side hybrid quicksort of csrc/qsort.cuh: sampled
multi-pivot partition levels over a device work queue, then a CTA-local
partition plus the bitonic network on every range <= sort_bound.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

from ._lib import VX_SORT_GRAPH, SortConfigC, SortStatsC, check, lib
from ._region import check_kv, check_region, dev_ptr, host_ptr, on_device, stream_of, workspace
from .lanes import get_backend, is_device

__all__ = ["SortConfig", "sort", "sort_with_config", "sort_into", "select_pivot", "MAX_PACKS"]

MAX_PACKS = 16  # smallsort.py:40
_PIVOT_STRATEGIES = ("median3", "middle", "random")
_U64 = (1 << 64) - 1


@dataclass(frozen=True)
class SortConfig:
    """Tuning knobs (quicksort.py:28-46).

    sort_bound: largest range handed to the bitonic network (default
    16*lanes: 256 int32 / 128 float64; must not exceed it).  pivot_strategy
    is validated like the reference's and selects how the device levels draw
    the sample their pivots come from (a level takes up to 255 pivots at
    once): "median3" stratified hashed positions, "middle" stratum
    midpoints, "random" the reference's MMIX LCG seeded by pivot_seed
    (csrc/qsort.cuh sample_pos).  The sorted output is unique, so the
    strategy cannot change it.  skip_empty_stores / swap_buffered are CPU
    store-pattern options of the reference partition and are accepted as
    no-ops.
    """

    sort_bound: int | None = None
    pivot_strategy: str = "median3"
    skip_empty_stores: bool = False
    swap_buffered: bool = False
    backend: str = "auto"
    pivot_seed: int = 0

    def __post_init__(self):
        if self.pivot_strategy not in _PIVOT_STRATEGIES:
            raise ValueError(f"unknown pivot strategy {self.pivot_strategy!r}")


def _resolve_bound(config: SortConfig, lanes: int) -> int:
    bound = config.sort_bound if config.sort_bound is not None else MAX_PACKS * lanes
    assert 1 <= bound <= MAX_PACKS * lanes, "sort_bound exceeds small-sort capacity"
    return bound


def select_pivot(region, lo: int, hi: int, strategy: str = "median3", lcg_state: int | None = None) -> int:
    """Index of the pivot for the inclusive range [lo, hi] (quicksort.py:55-74).
    Host-side helper (reads at most three elements), used e.g. to pick the
    config-3 pivot."""
    assert lo <= hi
    if strategy == "middle":
        return (lo + hi) // 2
    if strategy == "random":
        state = (lcg_state if lcg_state is not None else 0) & _U64
        return lo + state % (hi - lo + 1)
    mid = (lo + hi) // 2
    a, b, c = (region[i].item() if hasattr(region[i], "item") else region[i] for i in (lo, mid, hi))
    if b <= a <= c or c <= a <= b:
        return lo
    if a <= b <= c or c <= b <= a:
        return mid
    return hi


def _cfg(config: SortConfig, bound: int, flags: int = 0) -> SortConfigC:
    return SortConfigC(bound, _PIVOT_STRATEGIES.index(config.pivot_strategy), int(config.skip_empty_stores),
                       int(config.swap_buffered), flags, int(config.pivot_seed) & _U64)


def sort_with_config(region, config: SortConfig) -> None:
    """Sort a region ascending in place under an explicit configuration."""
    n = len(region)
    if n < 2:
        return
    kind = check_region(region)
    backend = get_backend(config.backend, kind)
    bound = _resolve_bound(config, backend.lanes)
    L = lib()
    if is_device(region):
        _device_sort(kind, region, None, region, None, config, bound, True, "sort")
        return
    check(L.vx_host_quicksort(kind.code, host_ptr(region), n, backend.lanes, bound,
                              _PIVOT_STRATEGIES.index(config.pivot_strategy), int(config.skip_empty_stores),
                              int(config.swap_buffered), int(config.pivot_seed) & _U64), "sort")


def _device_sort(kind, src, values, out, out_values, config, bound, check_status, what, stats=None):
    """vx_sort_into on src's device and current stream; with check_status the
    stream is synchronised once at the end and device-side errors raise."""
    L = lib()
    n = len(src)
    with on_device(src):
        ws = workspace(L.vx_sort_workspace_bytes(kind.code, int(values is not None), n), src.device)
        # a call that promises no host synchronisation replays a CUDA graph from the first call on
        cfg = _cfg(config, bound, VX_SORT_GRAPH if not check_status and stats is None else 0)
        st = stream_of(src)
        check(L.vx_sort_into(kind.code, dev_ptr(src), dev_ptr(values) if values is not None else None,
                             dev_ptr(out), dev_ptr(out_values) if out_values is not None else None, n,
                             ctypes.byref(cfg), dev_ptr(ws), ws.numel(), st), what)
        if check_status or stats is not None:
            s = SortStatsC()
            check(L.vx_sort_status(dev_ptr(ws), n, st, ctypes.byref(s)), what)
            if stats is not None:
                stats.update({f: getattr(s, f) for f, _ in SortStatsC._fields_ if f != "reserved"})
    return out


def sort_into(src, out, config: SortConfig | None = None, values=None, out_values=None, *, check: bool = True,
              stats: dict | None = None):
    """Device-only out-of-place sort: out = sorted(src) (pairs with values /
    out_values).  src is only read, by the first partition level, so this
    costs the same HBM traffic as the in-place sort.  check=False keeps the
    call fully stream-ordered (no synchronisation; capturable into a CUDA
    graph) and skips the device error check; `stats` (a dict) receives the
    level / launch counters of the sort (synchronises)."""
    config = config or SortConfig()
    kind = check_region(src)
    assert is_device(src) and is_device(out), "sort_into takes CUDA tensors"
    check_region(out)
    assert out.dtype == src.dtype and len(out) == len(src) and out.device == src.device
    assert (values is None) == (out_values is None), "values and out_values go together"
    if values is not None:
        check_kv(src, values)
        check_kv(out, out_values)
    backend = get_backend(config.backend, kind)
    bound = _resolve_bound(config, backend.lanes)
    if len(src) == 0:
        return out
    return _device_sort(kind, src, values, out, out_values, config, bound, check, "sort_into", stats)


def sort_many(regions, config: SortConfig | None = None, out=None) -> None:
    """Sort a sequence of HOST regions (numpy arrays / CPU tensors), each
    ascending in place -- ``for r in regions: sort(r, config)`` with the
    copies pipelined: while one region's sorted keys travel back over PCIe
    the next region's input is already on its way in (two device slots,
    ``vx_host_sort_submit`` / ``vx_host_sort_wait``).  ``out`` (optional, same
    shapes) receives the sorted copies and leaves ``regions`` untouched.
    Page-locked regions (``tensor.pin_memory()``) are needed for the overlap;
    pageable ones give the same result at ``sort``'s speed."""
    config = config or SortConfig()
    regions = list(regions)
    outs = regions if out is None else list(out)
    assert len(outs) == len(regions), "out must match regions"
    L = lib()
    pending: list[int] = []
    for src, dst in zip(regions, outs):
        kind = check_region(src)
        assert not is_device(src) and not is_device(dst), "sort_many takes host regions; use sort() for CUDA tensors"
        if dst is not src:
            assert check_region(dst) is kind and len(dst) == len(src), "out region must match its source"
        backend = get_backend(config.backend, kind)
        bound = _resolve_bound(config, backend.lanes)
        if len(pending) == 2:
            check(L.vx_host_sort_wait(pending.pop(0)), "sort_many")
        t = ctypes.c_int(-1)
        check(L.vx_host_sort_submit(kind.code, host_ptr(src), None, host_ptr(dst), None, len(src), backend.lanes,
                                    bound, _PIVOT_STRATEGIES.index(config.pivot_strategy),
                                    int(config.pivot_seed) & _U64, ctypes.byref(t)), "sort_many")
        pending.append(t.value)
    for t in pending:
        check(L.vx_host_sort_wait(t), "sort_many")


def sort(region, config: SortConfig | None = None) -> None:
    """Sort a region of int32 or float64 ascending, in place (quicksort.py:137-143).
    NaN elements are unsupported."""
    sort_with_config(region, config or SortConfig())
