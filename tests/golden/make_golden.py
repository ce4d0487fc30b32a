"""Generate golden fixtures by running the REFERENCE implementation.

Run in the authoring container only (the reference is not present on the GPU
box); the outputs (``*.npz``) are committed next to this script:

    python tests/golden/make_golden.py

The reference package is imported from a copy under ``baseline/_ref``
(git-ignored), never from /root/reference directly, because numba writes
cache files next to the sources (finding 9).  Its native
(numba) backend is the reference's default ``auto`` path; the emulated
backend is the executable specification and is used where cheap to confirm
the two agree.

Fixtures written:

* ``sort_cases.npz``       -- reference ``sort`` outputs: Fig. 1 KAT, the
  test_quicksort size sweep (test_quicksort.py:57-66), adversarial patterns
  (test_quicksort.py:69-82), sentinel-heavy inputs; both kinds.
* ``partition_cases.npz``  -- reference ``partition_region`` outputs (full
  partitioned LAYOUT and boundary) for random sizes / pivots / flags.
* ``kv_cases.npz``         -- reference ``kv_sort`` and ``kv_partition_region``
  outputs, including the exact value order among duplicate keys.
* ``smallsort_cases.npz``  -- reference ``sort_small_region`` for every length
  1..16*L with the sentinel mixed in (test_smallsort.py:153-163).
* ``config_digests.json``  -- blake2b digests of reference outputs on the
  BASELINE configs at reduced sizes (inputs regenerated from their seeds).
"""

from __future__ import annotations

import hashlib
import json
import os
import shutil
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src/vexsort"
REF_COPY = os.path.join(REPO, "baseline", "_ref")

sys.path.insert(0, HERE)
import inputs  # noqa: E402  (seeded generators shared with the tests)


def import_reference():
    dst = os.path.join(REF_COPY, "vexsort")
    if not os.path.isdir(dst):
        os.makedirs(REF_COPY, exist_ok=True)
        shutil.copytree(REF_SRC, dst)
    # the reference's own tests, run through integration/_kernels_b200.py by
    # tests/test_gpu_integration.py (baseline/_ref is git-ignored; it travels
    # to the GPU box with the working tree)
    tdst = os.path.join(REF_COPY, "tests")
    if not os.path.isdir(tdst):
        shutil.copytree(os.path.join(os.path.dirname(os.path.dirname(REF_SRC)), "tests"), tdst)
    sys.path.insert(0, REF_COPY)
    import vexsort  # noqa: F401

    assert vexsort.native_available(), "reference native backend unavailable"
    return vexsort


def digest(*arrs) -> str:
    h = hashlib.blake2b(digest_size=16)
    for a in arrs:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def random_region(rng, dtype, n, lo=None, hi=None):
    # conftest.py:35-42 of the reference
    if dtype == np.int32:
        lo = -(2**31) if lo is None else lo
        hi = 2**31 - 1 if hi is None else hi
        return rng.integers(lo, hi, size=n, dtype=np.int64, endpoint=True).astype(np.int32)
    lo = -1e9 if lo is None else lo
    hi = 1e9 if hi is None else hi
    return rng.uniform(lo, hi, size=n)


def main():
    vx = import_reference()
    from vexsort.quicksort import SortConfig

    out = {}
    # ---------------------------------------------------------------- sort
    idx = 0
    for dt, tag in ((np.int32, "i32"), (np.float64, "f64")):
        cases = [np.array([3, 1, 2, 0, 5], dtype=dt)]  # Fig. 1 KAT
        rng = np.random.default_rng(1)
        sizes = rng.integers(0, 3000, size=40).tolist() + [0, 1, 2, 255, 256, 257]
        for n in sizes:
            cases.append(random_region(rng, dt, int(n)))
        n = 1 << 12
        cases.append(np.arange(n).astype(dt))
        cases.append(np.arange(n)[::-1].copy().astype(dt))
        cases.append(np.tile(np.arange(37), n // 37 + 1)[:n].astype(dt))
        cases.append(np.random.default_rng(5).integers(0, 8, size=n).astype(dt))
        # sentinel / extreme values present (pad-safety)
        r = random_region(np.random.default_rng(77), dt, 1000, -50, 50)
        r[::7] = np.iinfo(np.int32).max if dt == np.int32 else np.inf
        if dt == np.int32:
            r[3::11] = np.iinfo(np.int32).min
        else:
            r[3::11] = -np.inf
        cases.append(r)
        for c in cases:
            # all three pivot strategies must give the one sorted output
            outs = []
            for strategy in ("median3", "middle", "random"):
                a = c.copy()
                vx.sort(a, SortConfig(pivot_strategy=strategy, pivot_seed=9))
                outs.append(a)
            assert all(np.array_equal(o, outs[0]) for o in outs)
            assert np.array_equal(outs[0], np.sort(c))
            out[f"{tag}_{idx}_in"] = c
            out[f"{tag}_{idx}_out"] = outs[0]
            idx += 1
    np.savez_compressed(os.path.join(HERE, "sort_cases.npz"), **out)
    print("sort cases", len(out) // 2)

    # ----------------------------------------------------------- partition
    out = {}
    idx = 0
    for dt, tag in ((np.int32, "i32"), (np.float64, "f64")):
        rng = np.random.default_rng(42)
        for rep in range(160):
            n = int(rng.integers(0, 1200)) if rep < 150 else int(rng.integers(4000, 9000))
            arr = random_region(rng, dt, n, lo=-100, hi=100)
            pivot = int(rng.integers(-110, 110))
            if dt == np.float64 and rep % 3 == 0:
                pivot = float(pivot) + 0.5
            opt_a, opt_b = bool(rep & 1), bool(rep & 2)
            a = arr.copy()
            b = vx.partition_region(a, pivot, skip_empty_stores=opt_a, swap_buffered=opt_b)
            out[f"{tag}_{idx}_in"] = arr
            out[f"{tag}_{idx}_out"] = a
            out[f"{tag}_{idx}_meta"] = np.array([b, opt_a, opt_b], dtype=np.int64)
            out[f"{tag}_{idx}_pivot"] = np.array([pivot], dtype=np.float64)
            idx += 1
    np.savez_compressed(os.path.join(HERE, "partition_cases.npz"), **out)
    print("partition cases", idx)

    # ------------------------------------------------------------------ kv
    out = {}
    idx = 0
    for kdt, vdt, tag in ((np.int32, np.int32, "i32"), (np.float64, np.int64, "f64")):
        rng = np.random.default_rng(2024)
        for rep in range(40):
            n = int(rng.integers(0, 2500)) if rep < 37 else int(rng.integers(6000, 9000))
            span = [10, 1000, 2**31 - 1][rep % 3]
            keys = rng.integers(-span, span, size=n).astype(kdt)
            vals = np.arange(n, dtype=vdt)
            k, v = keys.copy(), vals.copy()
            vx.kv_sort(k, v)
            out[f"sort_{tag}_{idx}_kin"] = keys
            out[f"sort_{tag}_{idx}_kout"] = k
            out[f"sort_{tag}_{idx}_vout"] = v
            pivot = int(rng.integers(-span, span))
            k, v = keys.copy(), vals.copy()
            b = vx.kv_partition_region(k, v, pivot)
            out[f"part_{tag}_{idx}_kout"] = k
            out[f"part_{tag}_{idx}_vout"] = v
            out[f"part_{tag}_{idx}_meta"] = np.array([b, pivot], dtype=np.int64)
            idx += 1
    np.savez_compressed(os.path.join(HERE, "kv_cases.npz"), **out)
    print("kv cases", idx)

    # ------------------------------------------------------------ smallsort
    out = {}
    for dt, tag, cap, sent in ((np.int32, "i32", 256, 2**31 - 1), (np.float64, "f64", 128, np.inf)):
        rng = np.random.default_rng(7)
        for n in range(1, cap + 1):
            region = random_region(rng, dt, n, lo=-50, hi=50)
            if n >= 3:
                region[rng.integers(0, n)] = sent
            a = region.copy()
            vx.sort_small_region(a)
            out[f"{tag}_{n}_in"] = region
            out[f"{tag}_{n}_out"] = a
    np.savez_compressed(os.path.join(HERE, "smallsort_cases.npz"), **out)
    print("smallsort cases", len(out) // 2)

    # ------------------------------------------------ config digests (reduced)
    dig = {}
    # C1 at full size (2^20), bound 256
    x = inputs.c1_input()
    a = x.copy()
    vx.sort(a)
    dig["c1_i32_2^20"] = {"in": digest(x), "out": digest(a)}
    # C2 reduced: 2^12 segments
    from vexsort import _kernels

    for tag, dt in (("i32", np.int32), ("f64", np.float64)):
        offs, vals = inputs.c2_input(dt, nseg=1 << 12)
        a = vals.copy()
        sent = 2**31 - 1 if tag == "i32" else np.inf
        for s in range(len(offs) - 1):
            lo, hi = int(offs[s]), int(offs[s + 1])
            if tag == "i32" or hi - lo <= 128:
                vx.sort_small_region(a[lo:hi])
            else:
                _kernels.smallsort_region(a, lo, hi - lo, sent)
        dig[f"c2_{tag}_2^12seg"] = {"in": digest(offs, vals), "out": digest(a)}
    # C3 reduced: 2^20 f64 standard normal, median3 pivot
    x = inputs.c3_input(n=1 << 20)
    from vexsort.quicksort import select_pivot

    pivot = x[select_pivot(x, 0, len(x) - 1, "median3")]
    a = x.copy()
    b = vx.partition_region(a, pivot)
    dig["c3_f64_2^20"] = {"in": digest(x), "pivot": float(pivot), "split": int(b),
                          "layout": digest(a), "sorted_low": digest(np.sort(a[:b])),
                          "sorted_high": digest(np.sort(a[b:]))}
    # C4 reduced: 2^18 pairs
    k0, v0 = inputs.c4_input(n=1 << 18)
    k, v = k0.copy(), v0.copy()
    vx.kv_sort(k, v)
    dig["c4_kv_2^18"] = {"in": digest(k0, v0), "keys": digest(k), "vals": digest(v)}
    # C5 reduced: 2^18, four distributions, both dtypes
    for dist in ("uniform", "sorted", "reverse", "few"):
        for dt, tag in ((np.int32, "i32"), (np.float64, "f64")):
            x = inputs.c5_input(dt, dist, n=1 << 16)
            a = x.copy()
            vx.sort(a)
            dig[f"c5_{tag}_{dist}_2^16"] = {"in": digest(x), "out": digest(a)}
    with open(os.path.join(HERE, "config_digests.json"), "w") as f:
        json.dump(dig, f, indent=1, sort_keys=True)
    print("digests", len(dig))


if __name__ == "__main__":
    main()
