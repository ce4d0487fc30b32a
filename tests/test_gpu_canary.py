"""Out-of-bounds and never-overwrite checks without a sanitizer.

compute-sanitizer is closed on this GPU pool (profiles/sanitizer_r2/), so the
memory-safety contract the reference pins (never write outside the region,
O(1) auxiliary space: pkg/tests/conftest.py:45-80, test_partition.py:183-209)
is checked the direct way: every buffer an operation may write -- keys,
payload, outputs AND the library's workspace -- sits between two guard zones
filled with a pattern, and the guards plus every read-only input must be
bit-identical afterwards.  tools/check_build.sh runs the same tests against
a -DVX_CHECK build whose kernels assert every bucket index, staging slot and
destination index on the device.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

GUARD = 4096  # bytes on each side
PATTERN = 0xA5


class Guarded:
    """A payload view of `nbytes` (aligned as torch allocates, shifted by
    `shift` bytes) between two guard zones."""

    def __init__(self, nbytes: int, shift: int = 0):
        self.raw = torch.full((GUARD + shift + nbytes + GUARD,), PATTERN, dtype=torch.uint8, device="cuda")
        self.lo = GUARD + shift
        self.hi = self.lo + nbytes

    def view(self, dtype):
        return self.raw[self.lo:self.hi].view(dtype)

    def intact(self) -> bool:
        return bool((self.raw[: self.lo] == PATTERN).all().item()) and bool(
            (self.raw[self.hi:] == PATTERN).all().item())


@pytest.fixture()
def guarded_workspace(monkeypatch):
    """Every workspace the package allocates gets guard zones too."""
    import paper_1704_08579_b200 as vx
    from paper_1704_08579_b200 import _region

    made = []

    def ws(nbytes, device):
        g = Guarded(max(int(nbytes), 256))
        made.append(g)
        return g.view(torch.uint8)

    for mod in (_region, vx.quicksort, vx.partition, vx.smallsort, vx.sharded):
        if hasattr(mod, "workspace"):
            monkeypatch.setattr(mod, "workspace", ws)
    return made


def _put(g: Guarded, a: np.ndarray):
    t = g.view(torch.from_numpy(a[:1]).dtype if a.size else torch.uint8)
    t.copy_(torch.from_numpy(a))
    return t


def _data(dt, n, kind, rng):
    if kind == "sorted":
        return (np.arange(n, dtype=np.int64) - n // 2).astype(dt)
    if kind == "few":
        return rng.integers(0, 16, n).astype(dt)
    if dt == np.int32:
        return rng.integers(-(2**31), 2**31 - 1, n, dtype=np.int32, endpoint=True)
    return rng.uniform(-1e6, 1e6, n)


SIZES = [1, 2, 255, 257, 8193, (1 << 16) + 5, (1 << 20) + 3, (1 << 24) + 7]


@pytest.mark.parametrize("dt", [np.int32, np.float64])
@pytest.mark.parametrize("kind", ["uniform", "sorted", "few"])
def test_sort_in_place_and_into_stay_inside_their_buffers(dt, kind, guarded_workspace):
    import paper_1704_08579_b200 as vx

    rng = np.random.default_rng(5)
    for n in SIZES:
        for shift in (0, dt().itemsize):  # aligned and element-misaligned views
            x = _data(dt, n, kind, rng)
            g = Guarded(x.nbytes, shift)
            t = _put(g, x)
            vx.sort(t)
            torch.cuda.synchronize()
            assert np.array_equal(t.cpu().numpy(), np.sort(x)), (n, shift)
            assert g.intact(), ("sort wrote outside its region", n, shift)
            # out of place: the input is never written
            gi, go = Guarded(x.nbytes, shift), Guarded(x.nbytes)
            ti, to = _put(gi, x), go.view(t.dtype)
            vx.sort_into(ti, to)
            torch.cuda.synchronize()
            assert np.array_equal(ti.cpu().numpy(), x), ("sort_into overwrote its input", n)
            assert np.array_equal(to.cpu().numpy(), np.sort(x))
            assert gi.intact() and go.intact()
    assert guarded_workspace and all(w.intact() for w in guarded_workspace), "workspace overrun"


@pytest.mark.parametrize("kdt,vdt", [(np.int32, np.int32), (np.float64, np.int64)])
def test_kv_sort_stays_inside_its_buffers(kdt, vdt, guarded_workspace):
    import paper_1704_08579_b200 as vx

    rng = np.random.default_rng(6)
    for n in (1, 300, 8200, (1 << 18) + 1, (1 << 23) + 9):
        k = _data(kdt, n, "uniform", rng) if kdt == np.float64 else rng.integers(0, 2**31 - 1, n, dtype=np.int32)
        v = np.arange(n, dtype=vdt)
        gk, gv = Guarded(k.nbytes), Guarded(v.nbytes, v.itemsize)
        tk, tv = _put(gk, k), _put(gv, v)
        vx.kv_sort(tk, tv)
        torch.cuda.synchronize()
        ko, vo = tk.cpu().numpy(), tv.cpu().numpy()
        assert np.array_equal(ko, np.sort(k)) and np.array_equal(k[vo], ko)
        assert np.array_equal(np.sort(vo), v)
        assert gk.intact() and gv.intact(), n
    assert all(w.intact() for w in guarded_workspace)


@pytest.mark.parametrize("dt", [np.int32, np.float64])
def test_partition_stays_inside_its_buffers(dt, guarded_workspace):
    import paper_1704_08579_b200 as vx

    rng = np.random.default_rng(7)
    for n in (1, 2, 1000, 4097, (1 << 20) + 11, (1 << 24) + 1):
        for shift in (0, dt().itemsize):
            x = _data(dt, n, "uniform", rng)
            piv = x[n // 2]
            g = Guarded(x.nbytes, shift)
            t = _put(g, x)
            b = vx.partition_region(t, piv)
            torch.cuda.synchronize()
            got = t.cpu().numpy()
            assert b == int(np.count_nonzero(x <= piv))
            assert np.all(got[:b] <= piv) and np.all(got[b:] > piv)
            assert np.array_equal(np.sort(got), np.sort(x))
            assert g.intact(), (n, shift)
    assert all(w.intact() for w in guarded_workspace)


@pytest.mark.parametrize("dt", [np.int32, np.float64])
def test_segment_sort_stays_inside_its_buffers(dt, guarded_workspace):
    import paper_1704_08579_b200 as vx

    rng = np.random.default_rng(8)
    lens = rng.integers(1, 257, size=5000)
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    x = _data(dt, int(offs[-1]), "uniform", rng)
    g, go = Guarded(x.nbytes, x.itemsize), Guarded(offs.nbytes)
    t, o = _put(g, x), _put(go, offs)
    vx.sort_segments(t, o)
    torch.cuda.synchronize()
    got = t.cpu().numpy()
    for i in range(len(lens)):
        assert np.array_equal(got[offs[i]:offs[i + 1]], np.sort(x[offs[i]:offs[i + 1]]))
    assert np.array_equal(o.cpu().numpy(), offs), "offsets were written"
    assert g.intact() and go.intact()
    assert all(w.intact() for w in guarded_workspace)
