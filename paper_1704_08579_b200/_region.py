"""Region plumbing shared by the API modules: validation, workspace, stream,
pivot conversion.  No compute happens here."""

from __future__ import annotations

import ctypes
import math

import numpy as np

from .lanes import ElemKind, kind_of, is_device

__all__ = ["check_region", "check_kv", "workspace", "stream_of", "pivot_for", "host_ptr", "dev_ptr", "on_device"]


def check_region(region) -> ElemKind:
    kind = kind_of(region)
    if region.ndim != 1:
        raise AssertionError("regions are 1-D")
    contiguous = region.is_contiguous() if is_device(region) or hasattr(region, "is_contiguous") \
        else region.flags.c_contiguous
    if not contiguous:
        raise AssertionError("regions must be contiguous")
    return kind


def check_kv(keys, values) -> ElemKind:
    """keyvalue.py:44-47 -- same length, same element width, same device."""
    kind = check_region(keys)
    if values.ndim != 1:
        raise AssertionError("regions are 1-D")
    assert len(keys) == len(values), "keys and values must have equal length"
    assert _itemsize(keys) == _itemsize(values), "values must have the same element width as keys"
    assert is_device(keys) == is_device(values), "keys and values must live on the same device"
    if is_device(keys):
        assert keys.device == values.device, "keys and values must live on the same device"
        assert values.is_contiguous(), "regions must be contiguous"
    elif hasattr(values, "flags"):
        assert values.flags.c_contiguous, "regions must be contiguous"
    return kind


def _itemsize(a) -> int:
    if hasattr(a, "element_size"):
        return a.element_size()
    return a.dtype.itemsize


def workspace(nbytes: int, device):
    import torch

    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


def on_device(t):
    """Make t's GPU the current device for the duration of a C-ABI call (the
    library runs on the current device; its per-device state follows it)."""
    import torch

    return torch.cuda.device(t.device)


def stream_of(t) -> ctypes.c_void_p:
    import torch

    return ctypes.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def dev_ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


def host_ptr(a) -> ctypes.c_void_p:
    """Address of a host region (numpy array or CPU tensor)."""
    if isinstance(a, np.ndarray):
        return ctypes.c_void_p(a.ctypes.data)
    return ctypes.c_void_p(a.data_ptr())


def pivot_for(kind: ElemKind, pivot):
    """Convert a Python pivot to the key type with the reference's
    mathematical comparison semantics (numba compares int32 against a float
    pivot exactly).  Returns (ctypes scalar, shortcut) where shortcut is
    "none" (nothing is <= pivot), "all" (everything is) or None."""
    if hasattr(pivot, "item") and not isinstance(pivot, (int, float)):
        pivot = pivot.item()  # numpy / torch scalars
    if kind.name == "f64":
        return ctypes.c_double(float(pivot)), None
    p = int(pivot) if isinstance(pivot, (int, np.integer)) else float(pivot)
    if isinstance(p, float):
        if math.isnan(p):
            return None, "none"
        if math.isinf(p):
            return None, "all" if p > 0 else "none"
        p = math.floor(p)
    p = int(p)
    if p < -(2**31):
        return None, "none"
    if p >= 2**31 - 1:
        return ctypes.c_int32(2**31 - 1), None
    return ctypes.c_int32(p), None
