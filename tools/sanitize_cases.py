"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every kernel family of the library on sizes that reach each
code path (finish-only, global levels + finish, the CTA-local level), with
the results checked against numpy so a run also proves correctness under
the tool.  Used by tools/sanitize.sh on the GPU box.

    python tools/sanitize_cases.py [quick|full]
"""

from __future__ import annotations

import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1704_08579_b200 as vx  # noqa: E402

dev = torch.device("cuda:0")
rng = np.random.default_rng(7)
mode = sys.argv[1] if len(sys.argv) > 1 else "full"


def rand(dt, n, kind="uniform"):
    if kind == "sorted":
        a = np.arange(n, dtype=np.int64) - n // 2
        return a.astype(dt)
    if kind == "few":
        return rng.integers(0, 16, n).astype(dt)
    if dt == np.int32:
        return rng.integers(-(2**31), 2**31 - 1, n, dtype=np.int32, endpoint=True)
    return rng.uniform(-1e6, 1e6, n)


def check_sort(dt, n, kind="uniform"):
    x = rand(dt, n, kind)
    t = torch.from_numpy(x).to(dev)
    vx.sort(t)
    assert np.array_equal(t.cpu().numpy(), np.sort(x)), (dt, n, kind)
    print(f"sort {np.dtype(dt).name} n={n} {kind}: ok", flush=True)


def check_kv(dt, n):
    k = rand(dt, n)
    v = np.arange(n, dtype=np.int32 if dt == np.int32 else np.int64)
    tk, tv = torch.from_numpy(k).to(dev), torch.from_numpy(v).to(dev)
    vx.kv_sort(tk, tv)
    gk, gv = tk.cpu().numpy(), tv.cpu().numpy()
    assert np.array_equal(gk, np.sort(k)) and np.array_equal(k[gv], gk)
    print(f"kv {np.dtype(dt).name} n={n}: ok", flush=True)


def check_partition(n, offset=0):
    y = rng.standard_normal(n + offset)
    t = torch.from_numpy(y).to(dev)[offset:]
    piv = float(np.median(y[offset:]))
    b = vx.partition_region(t, piv)
    got = t.cpu().numpy()
    assert b == int((y[offset:] <= piv).sum()) and np.all(got[:b] <= piv) and np.all(got[b:] > piv)
    print(f"partition n={n} offset={offset}: ok", flush=True)


def check_segments(nseg):
    lens = rng.integers(1, 257, nseg)
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    x = rand(np.int32, int(offs[-1]))
    t = torch.from_numpy(x).to(dev)
    vx.sort_segments(t, torch.from_numpy(offs).to(dev))
    got = t.cpu().numpy()
    for s in range(0, nseg, max(1, nseg // 64)):
        assert np.array_equal(got[offs[s]:offs[s + 1]], np.sort(x[offs[s]:offs[s + 1]]))
    print(f"segments nseg={nseg}: ok", flush=True)


def check_bucket_partition(n):
    from paper_1704_08579_b200.sharded import B200Ops

    ops = B200Ops()
    x = torch.from_numpy(rand(np.int32, n)).to(dev)
    gi = torch.arange(n, dtype=torch.int64, device=dev)
    pos = torch.linspace(0, n - 1, 512).long().to(dev)
    sk, si = ops.select_splitters(x[pos].contiguous(), gi[pos].contiguous(), 8)
    out, counts = ops.bucket_partition(x, 0, sk, si)
    assert int(counts.sum()) == n
    assert np.array_equal(np.sort(out.cpu().numpy()), np.sort(x.cpu().numpy()))
    print(f"bucket_partition n={n}: ok", flush=True)


check_sort(np.int32, 1 << 12)
check_sort(np.float64, 5000)
check_sort(np.int32, 1 << 20)
check_sort(np.int32, 1 << 20, "sorted")
check_sort(np.int32, 1 << 20, "few")
check_kv(np.int32, 1 << 18)
check_partition(1 << 20)
check_partition(1 << 20, offset=1)
check_segments(4096)
check_bucket_partition(1 << 20)
if mode == "full":
    # the CTA-local level starts at 256 x its target (2^24 int32, 2^23 f64 / pairs)
    check_sort(np.float64, 1 << 20)
    check_sort(np.float64, 1 << 23)
    check_sort(np.int32, 1 << 24)
    check_kv(np.int32, 1 << 23)
torch.cuda.synchronize()
print("sanitize cases: all ok")
