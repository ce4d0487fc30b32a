"""Device-side output verification (the bench gate and the full-size parity
tests).

The reference gates every benchmark on "the output equals np.sort of the
input" (benchcli.py:398-427, exit 1 otherwise).  At 2^31-2^32 elements the
output cannot be brought home cheaply, so the gate is restated as
size-independent properties computed on the device by ``vx_verify``:

* the output is ascending (adjacent inversions == 0), and
* input and output hold the same multiset (sum and xor of a per-element
  hash agree; pairs hash key and value bits together).

For a total order on the keys (no NaN, no -0.0 -- the generators exclude
both) these two properties imply ``out == np.sort(in)`` bit for bit.
``positional`` is an order-dependent digest of an array, computed the same
way in numpy by tests/golden/make_full_digests.py, which pins the full-size
outputs to the oracle's.
"""

from __future__ import annotations

from dataclasses import dataclass

from ._lib import check, lib
from ._region import check_region, dev_ptr, stream_of

__all__ = ["Digest", "digest", "verify_sorted_permutation", "generate", "DISTS", "MASK64"]

MASK64 = (1 << 64) - 1


@dataclass(frozen=True)
class Digest:
    n: int
    hsum: int        # sum of per-element hashes mod 2^64 (order-independent)
    hxor: int        # xor of per-element hashes (order-independent)
    inversions: int  # adjacent k[i+1] < k[i] (within segments when offsets are given)
    positional: int  # sum of mix64(bits ^ mix64(i)) mod 2^64 (order-dependent)

    def multiset(self):
        return (self.n, self.hsum, self.hxor)


def digest(keys, values=None, *, order: bool = True, offsets=None) -> Digest:
    """Digest of a device array (and its payload); synchronises."""
    import torch

    kind = check_region(keys)
    assert keys.is_cuda, "digest takes CUDA tensors"
    if values is not None:
        assert values.is_cuda and len(values) == len(keys) and values.element_size() == keys.element_size()
    out = torch.zeros(4, dtype=torch.int64, device=keys.device)
    nseg = 0
    if offsets is not None:
        assert offsets.dtype == torch.int64 and offsets.is_cuda and offsets.is_contiguous()
        nseg = len(offsets) - 1
    with torch.cuda.device(keys.device):
        check(lib().vx_verify(kind.code, dev_ptr(keys), dev_ptr(values) if values is not None else None, len(keys),
                              int(order), dev_ptr(offsets) if offsets is not None else None, nseg, dev_ptr(out),
                              stream_of(keys)), "verify")
    s, x, inv, pos = (int(v) & MASK64 for v in out.cpu().tolist())
    return Digest(len(keys), s, x, inv, pos)


def verify_sorted_permutation(src, out, src_values=None, out_values=None, *, offsets=None) -> Digest:
    """Raise AssertionError unless `out` is `src` sorted ascending (per CSR
    segment when `offsets` is given; pairs carried along).  Returns the
    output digest."""
    d_in = digest(src, src_values, order=False)
    d_out = digest(out, out_values, order=True, offsets=offsets)
    assert d_out.inversions == 0, f"output not sorted: {d_out.inversions} adjacent inversions"
    assert d_in.multiset() == d_out.multiset(), "output is not a permutation of the input"
    return d_out


DISTS = {"uniform": 0, "sorted": 1, "reverse": 2, "few": 3, "normal": 4, "u31": 5, "index": 6}


def generate(dtype, dist: str, n: int, *, seed: int = 1, global_offset: int = 0, global_n: int | None = None,
             device=None):
    """Seeded synthetic input generated on the device (vx_generate: a counter
    hash of the global index, so every rank count P yields the same global
    array).  dtype: torch.int32 or torch.float64."""
    import torch

    device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    t = torch.empty(n, dtype=dtype, device=device)
    code = 0 if dtype == torch.int32 else 1
    with torch.cuda.device(device):
        check(lib().vx_generate(code, DISTS[dist], dev_ptr(t), n, seed, global_offset,
                                global_n if global_n is not None else n, stream_of(t)), "generate")
    return t
