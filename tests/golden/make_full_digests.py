"""Full-size golden digests (BASELINE configs 2 and 5 at their benchmarked
sizes), written to ``full_digests.json`` next to this script.

Run in the authoring container only (needs ~40 GB of RAM and the reference
copy for C2; minutes of CPU):

    python tests/golden/make_full_digests.py [c2] [c5]

* **C5** (int32 n = 2^32, float64 n = 2^31, four distributions).  The
  reference's correctness oracle for a full sort is ``np.sort``
  (pkg/src/vexsort/oracle.py:15-21; the reference's own quicksort is
  quadratic on three of the distributions and ~28 min on the fourth).  The
  inputs are the bench's DEVICE generator (``vx_generate``, a counter hash
  of the global index), replicated here in numpy bit for bit
  (``gen_numpy``); each input is sorted with ``np.sort`` and summarised by
  the same digests ``vx_verify`` computes on the device
  (paper_1704_08579_b200/verify.py): the order-independent multiset digest
  of the input and the order-dependent positional digest of ``np.sort``.
  A GPU test that reproduces the positional digest therefore holds the
  oracle's exact output at full size.
* **C2** (2^20 CSR segments, int32 and float64): the REFERENCE's own per
  segment small sort (``sort_small_region``, or ``_kernels.smallsort_region``
  for float64 segments longer than 16*L = 128) over the whole input, as a
  blake2b digest of the output (same scheme as config_digests.json).
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
OUT = os.path.join(HERE, "full_digests.json")

M64 = (1 << 64) - 1
U = np.uint64
DIST = {"uniform": 0, "sorted": 1, "reverse": 2, "few": 3}


def mix64(x):
    """splitmix64 finaliser (common.cuh mix64) on a uint64 array."""
    x = x + U(0x9E3779B97F4A7C15)
    x = (x ^ (x >> U(30))) * U(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> U(27))) * U(0x94D049BB133111EB)
    return x ^ (x >> U(31))


def gen_numpy(is_i32: bool, dist: str, g0: int, m: int, gn: int, seed: int = 1):
    """Elements [g0, g0+m) of vx_generate(dtype, dist, seed) (vexsort_b200.cu
    gen_kernel), bit for bit."""
    g = np.arange(g0, g0 + m, dtype=np.uint64)
    with np.errstate(over="ignore"):
        h = mix64(U((seed * 0xD1B54A32D192ED03) & M64) + g)
        step = U((1 << 32) // gn)
        if is_i32:
            if dist == "uniform":
                return (h >> U(32)).astype(np.uint32).view(np.int32)
            if dist == "sorted":
                return ((g * step - U(1 << 31)) & U(0xFFFFFFFF)).astype(np.uint32).view(np.int32)
            if dist == "reverse":
                return ((U(0x7FFFFFFF) - g * step) & U(0xFFFFFFFF)).astype(np.uint32).view(np.int32)
            return (h >> U(60)).astype(np.int32)
        if dist == "uniform":
            u = (h >> U(11)).astype(np.float64) * 2.0**-53
            return -1e6 + 2e6 * u  # two roundings, as __dadd_rn(__dmul_rn(...)) on the device
        if dist == "sorted":
            return g.astype(np.float64) - 1073741824.0
        if dist == "reverse":
            return 1073741823.0 - g.astype(np.float64)
        return (h >> U(60)).astype(np.float64)


def bits64(a):
    return a.view(np.uint32).astype(np.uint64) if a.dtype == np.int32 else a.view(np.uint64)


def digests(a, base: int, with_pos: bool):
    """(sum, xor, positional) partial digests of a chunk starting at global
    position `base`."""
    b = bits64(a)
    with np.errstate(over="ignore"):
        h = mix64(b)
        s = int(h.sum(dtype=np.uint64))
        x = int(np.bitwise_xor.reduce(h))
        p = 0
        if with_pos:
            i = np.arange(base, base + len(a), dtype=np.uint64)
            p = int((mix64(b ^ mix64(i))).sum(dtype=np.uint64))
    return s, x, p


def c5(results):
    CH = 1 << 26
    for tag, is_i32, n in (("i32", True, 1 << 32), ("f64", False, 1 << 31)):
        for dist in DIST:
            key = f"c5_{tag}_{dist}"
            if key in results:
                continue
            t0 = time.time()
            a = np.empty(n, dtype=np.int32 if is_i32 else np.float64)
            hs = hx = 0
            for c0 in range(0, n, CH):
                a[c0:c0 + CH] = gen_numpy(is_i32, dist, c0, CH, n)
                s, x, _ = digests(a[c0:c0 + CH], c0, False)
                hs, hx = (hs + s) & M64, hx ^ x
            if not is_i32:
                assert not np.isnan(a).any() and not np.any((a == 0) & np.signbit(a))
            a.sort()
            ps = 0
            for c0 in range(0, n, CH):
                _, _, p = digests(a[c0:c0 + CH], c0, True)
                ps = (ps + p) & M64
            results[key] = {"n": n, "dist_code": DIST[dist], "seed": 1, "hsum": hs, "hxor": hx, "sorted_positional": ps,
                            "first": a[0].item(), "last": a[-1].item()}
            del a
            print(key, f"{time.time() - t0:.0f}s", flush=True)
            save(results)


def c2(results):
    import hashlib

    sys.path.insert(0, os.path.dirname(HERE))
    from golden.make_golden import import_reference
    import inputs

    vx = import_reference()
    from vexsort import _kernels

    def dg(*arrs):
        h = hashlib.blake2b(digest_size=16)
        for x in arrs:
            h.update(np.ascontiguousarray(x).tobytes())
        return h.hexdigest()

    for tag, dt in (("i32", np.int32), ("f64", np.float64)):
        key = f"c2_{tag}_2^20seg"
        if key in results:
            continue
        t0 = time.time()
        offs, vals = inputs.c2_input(dt, nseg=1 << 20)
        a = vals.copy()
        sent = 2**31 - 1 if tag == "i32" else np.inf
        for s in range(len(offs) - 1):
            lo, hi = int(offs[s]), int(offs[s + 1])
            if tag == "i32" or hi - lo <= 128:
                vx.sort_small_region(a[lo:hi])
            else:
                _kernels.smallsort_region(a, lo, hi - lo, sent)
        # the reference agrees with np.sort segment by segment
        seg = np.repeat(np.arange(len(offs) - 1), np.diff(offs))
        assert np.array_equal(a, vals[np.lexsort((vals, seg))])
        results[key] = {"nseg": 1 << 20, "n": int(offs[-1]), "in": dg(offs, vals), "out": dg(a)}
        print(key, f"{time.time() - t0:.0f}s", flush=True)
        save(results)


def save(results):
    with open(OUT, "w") as f:
        json.dump(results, f, indent=1, sort_keys=True)


def main():
    results = json.load(open(OUT)) if os.path.exists(OUT) else {}
    what = sys.argv[1:] or ["c2", "c5"]
    if "c2" in what:
        c2(results)
    if "c5" in what:
        c5(results)


if __name__ == "__main__":
    main()
