"""Seeded host-side input generators for the five BASELINE configs.

Shared by tests/golden/make_golden.py (fixtures from the reference), the
parity tests and bench.py's CPU legs.  Streams follow SURVEY.md section 8(d):
``default_rng(SeedSequence([S, cfg, dtype_id, log2n, chunk]))`` with base
seed S = 1 (the reference bench default, benchcli.py:518), the benchcli
scheme (benchcli.py:81-97) plus a chunk id.  No generator emits NaN or -0.0
(asserted), so sorted outputs are unique bit patterns.
"""

from __future__ import annotations

import numpy as np

SEED = 1
_DT = {np.dtype(np.int32): 0, np.dtype(np.float64): 1}


def _rng(cfg: int, dtype, n: int, chunk: int = 0):
    log2n = int(n).bit_length() - 1
    ss = np.random.SeedSequence([SEED, cfg, _DT[np.dtype(dtype)], log2n, chunk])
    return np.random.default_rng(ss)


def _clean(x):
    if x.dtype == np.float64:
        assert not np.isnan(x).any()
        assert not np.any((x == 0) & np.signbit(x)), "-0.0 in generated input"
    return x


def c1_input(n: int = 1 << 20):
    """C1: int32 i.i.d. uniform over the full range (benchcli.py:91-92)."""
    rng = _rng(1, np.int32, n)
    return rng.integers(-(2**31), 2**31 - 1, size=n, dtype=np.int32, endpoint=True)


def c2_input(dtype, nseg: int = 1 << 20):
    """C2: CSR segments with lengths U{1..256}; int32 full range or f64
    uniform in [-1e6, 1e6).  Returns (offsets int64[nseg+1], values)."""
    rng = _rng(2, dtype, nseg)
    lens = rng.integers(1, 257, size=nseg)
    offs = np.zeros(nseg + 1, dtype=np.int64)
    np.cumsum(lens, out=offs[1:])
    n = int(offs[-1])
    if np.dtype(dtype) == np.int32:
        vals = rng.integers(-(2**31), 2**31 - 1, size=n, dtype=np.int32, endpoint=True)
    else:
        vals = rng.uniform(-1e6, 1e6, size=n)
    return offs, _clean(vals)


def c3_input(n: int = 1 << 28):
    """C3: f64 i.i.d. standard normal."""
    return _clean(_rng(3, np.float64, n).standard_normal(n))


def c4_input(n: int = 1 << 28):
    """C4: int32 keys uniform in [0, 2^31), int32 values = original index."""
    rng = _rng(4, np.int32, n)
    keys = rng.integers(0, 2**31, size=n, dtype=np.int32)
    return keys, np.arange(n, dtype=np.int32)


def c5_chunk(dtype, dist: str, n: int, chunk: int, nchunks: int = 64):
    """One of the 64 fixed chunks of the C5 global input (so the global
    array is identical for every rank count P)."""
    assert n % nchunks == 0
    m = n // nchunks
    base = chunk * m
    i = np.arange(base, base + m, dtype=np.int64)
    is_i32 = np.dtype(dtype) == np.int32
    if dist == "uniform":
        rng = _rng(5, dtype, n, chunk)
        if is_i32:
            return rng.integers(-(2**31), 2**31 - 1, size=m, dtype=np.int32, endpoint=True)
        return _clean(rng.uniform(-1e6, 1e6, size=m))
    if dist == "sorted":
        return (i - 2**31).astype(np.int32) if is_i32 else _clean(i.astype(np.float64) - 2.0**30)
    if dist == "reverse":
        return (2**31 - 1 - i).astype(np.int32) if is_i32 else _clean(2.0**30 - 1 - i.astype(np.float64))
    if dist == "few":
        rng = _rng(5, dtype, n, chunk)
        x = rng.integers(0, 16, size=m)
        return x.astype(np.int32) if is_i32 else x.astype(np.float64)
    raise ValueError(dist)


def c5_input(dtype, dist: str, n: int, rank: int = 0, world: int = 1, nchunks: int = 64):
    """Rank `rank`'s contiguous share (chunks [64r/P, 64(r+1)/P)) of the C5
    global input of n elements."""
    c0, c1 = nchunks * rank // world, nchunks * (rank + 1) // world
    return np.concatenate([c5_chunk(dtype, dist, n, c, nchunks) for c in range(c0, c1)])
