"""Element kinds and the backend registry (mirror of vexsort/lanes.py).

The reference's plugin point is the backend object returned by
``get_backend(name, kind)`` (lanes.py:483-499); region algorithms route to
the native kernels whenever ``backend.uses_kernels`` (lanes.py:297).  Here
there is exactly one backend, the B200 one: "auto", "native" and "b200" all
resolve to it.  The reference's CPU lane emulation ("emulated") is not part
of this build (no CPU fallback) and raises :class:`BackendUnavailable`.

Regions are 1-D contiguous arrays: ``torch`` CUDA tensors run on the device
directly; numpy arrays and CPU tensors take the host-buffer path (copy to the
B200, sort there, copy back in place), which is what the reference's callers
pass today.
"""

from __future__ import annotations

import math
from typing import NamedTuple

import numpy as np

from ._lib import VX_F64, VX_I32, BackendUnavailable, lib

__all__ = [
    "ElemKind",
    "I32",
    "F64",
    "KINDS",
    "BackendUnavailable",
    "B200Backend",
    "get_backend",
    "available_backends",
    "native_available",
    "native_unavailable_reason",
    "has_full_width_vectors",
    "kind_of",
    "is_device",
]


class ElemKind(NamedTuple):
    """An element kind with the reference's lane geometry and sentinel
    (lanes.py:50-63).  `code` is the C-ABI dtype code."""

    name: str
    dtype: np.dtype
    lanes: int
    sentinel: int | float
    py: type
    code: int


I32 = ElemKind("i32", np.dtype(np.int32), 16, 2**31 - 1, int, VX_I32)
F64 = ElemKind("f64", np.dtype(np.float64), 8, math.inf, float, VX_F64)
KINDS = {"i32": I32, "f64": F64}


def _torch():
    import torch

    return torch


def is_device(region) -> bool:
    """True for a CUDA torch tensor (device path)."""
    try:
        torch = _torch()
    except ImportError:  # pragma: no cover
        return False
    return isinstance(region, torch.Tensor) and region.is_cuda


def kind_of(region) -> ElemKind:
    """Element kind by dtype; TypeError otherwise (lanes.py:502-507)."""
    dt = getattr(region, "dtype", None)
    try:
        torch = _torch()
        if isinstance(region, torch.Tensor):
            if dt == torch.int32:
                return I32
            if dt == torch.float64:
                return F64
            raise TypeError(f"unsupported element dtype {dt}; use int32 or float64")
    except ImportError:  # pragma: no cover
        pass
    for kind in KINDS.values():
        if np.dtype(dt) == kind.dtype:
            return kind
    raise TypeError(f"unsupported element dtype {dt}; use int32 or float64")


class B200Backend:
    """The one backend of this build: sm_100a kernels behind the C ABI."""

    name = "b200"
    uses_kernels = True

    def __init__(self, kind: ElemKind):
        self.kind = kind
        self.lanes = kind.lanes

    def __repr__(self):
        return f"B200Backend({self.kind.name})"


def _probe() -> str | None:
    try:
        lib()
    except BackendUnavailable as exc:
        return str(exc)
    try:
        torch = _torch()
        if not torch.cuda.is_available():
            return "no CUDA device visible"
    except ImportError as exc:  # pragma: no cover
        return f"torch unavailable: {exc}"
    return None


def native_unavailable_reason() -> str | None:
    return _probe()


def native_available() -> bool:
    return _probe() is None


def has_full_width_vectors() -> bool:
    """Kept for API parity (lanes.py:422-429): the B200 path has no 512-bit
    CPU vector requirement."""
    return True


def available_backends() -> tuple[str, ...]:
    return ("b200",) if native_available() else ()


_CACHE: dict[tuple[str, str], B200Backend] = {}


def get_backend(name: str, kind: ElemKind | str):
    """Backend `name` for `kind` ("auto" / "native" / "b200")."""
    if isinstance(kind, str):
        kind = KINDS[kind]
    if name not in ("auto", "native", "b200", "emulated"):
        raise ValueError(f"unknown backend {name!r}")
    if name == "emulated":
        raise BackendUnavailable("the CPU lane emulation is not part of the B200 build")
    key = ("b200", kind.name)
    be = _CACHE.get(key)
    if be is None:
        be = _CACHE[key] = B200Backend(kind)
    return be
