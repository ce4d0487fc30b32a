"""Pin the CPU oracle (oracle/vexsort_oracle.c) to fixtures produced by the
reference implementation itself (tests/golden/make_golden.py).

The oracle must reproduce the reference bit-for-bit, including the
partitioned LAYOUT (the reference's own emulated-vs-native bit-identity
contract, test_partition.py:84-101) and the kv value order among equal keys.
CPU-only: no GPU needed.
"""

import json
import os

import numpy as np
import pytest

import oracle
import inputs


def _load(golden_dir, name):
    return np.load(os.path.join(golden_dir, name))


def _cases(z, prefix=""):
    ids = sorted({k.rsplit("_", 1)[0] for k in z.files if k.startswith(prefix)})
    return ids


def test_sort_cases_match_reference(golden_dir):
    z = _load(golden_dir, "sort_cases.npz")
    n = 0
    for cid in _cases(z):
        x, want = z[cid + "_in"], z[cid + "_out"]
        for strategy in ("median3", "middle", "random"):
            a = x.copy()
            oracle.sort(a, pivot_strategy=strategy, seed=9)
            assert np.array_equal(a, want), (cid, strategy)
        n += 1
    assert n > 100


def test_sort_task_parallel_variant_identical(golden_dir):
    z = _load(golden_dir, "sort_cases.npz")
    for cid in _cases(z):
        x, want = z[cid + "_in"], z[cid + "_out"]
        a = x.copy()
        oracle.sort(a, nthreads=4)
        assert np.array_equal(a, want), cid


def test_partition_layouts_bit_identical_to_reference(golden_dir):
    z = _load(golden_dir, "partition_cases.npz")
    cnt = 0
    for cid in _cases(z):
        if not cid.endswith(tuple("0123456789")):
            continue
        x, want = z[cid + "_in"], z[cid + "_out"]
        b_want, opt_a, opt_b = (int(v) for v in z[cid + "_meta"])
        pivot = float(z[cid + "_pivot"][0])
        if x.dtype == np.int32:
            pivot = int(pivot)
        a = x.copy()
        b = oracle.partition_region(a, pivot, bool(opt_a), bool(opt_b))
        assert b == b_want, cid
        assert np.array_equal(a, want), cid
        # and the boundary is the count of <= pivot (numpy oracle.py twin)
        assert b == oracle.oracle_partition(x.copy(), pivot)
        cnt += 1
    assert cnt == 320


def test_kv_sort_and_partition_bit_identical_to_reference(golden_dir):
    z = _load(golden_dir, "kv_cases.npz")
    cnt = 0
    for tag, vdt in (("i32", np.int32), ("f64", np.int64)):
        for i in range(80):
            key = f"sort_{tag}_{i}"
            if key + "_kin" not in z.files:
                continue
            kin = z[key + "_kin"]
            k, v = kin.copy(), np.arange(len(kin), dtype=vdt)
            oracle.kv_sort(k, v)
            assert np.array_equal(k, z[key + "_kout"]), key
            assert np.array_equal(v, z[key + "_vout"]), key  # exact value order
            pk = f"part_{tag}_{i}"
            b_want, pivot = (int(t) for t in z[pk + "_meta"])
            k, v = kin.copy(), np.arange(len(kin), dtype=vdt)
            b = oracle.kv_partition_region(k, v, pivot)
            assert b == b_want
            assert np.array_equal(k, z[pk + "_kout"]) and np.array_equal(v, z[pk + "_vout"])
            cnt += 1
    assert cnt == 80


def test_smallsort_all_lengths_match_reference(golden_dir):
    z = _load(golden_dir, "smallsort_cases.npz")
    for cid in _cases(z):
        x, want = z[cid + "_in"], z[cid + "_out"]
        a = x.copy()
        oracle.smallsort_region(a, 0, len(a), oracle.sentinel_for(a))
        assert np.array_equal(a, want), cid


def test_config_digests_match_reference(golden_dir):
    from make_golden import digest

    with open(os.path.join(golden_dir, "config_digests.json")) as f:
        dig = json.load(f)
    x = inputs.c1_input()
    assert digest(x) == dig["c1_i32_2^20"]["in"]
    a = x.copy()
    oracle.sort(a)
    assert digest(a) == dig["c1_i32_2^20"]["out"]
    for tag, dt in (("i32", np.int32), ("f64", np.float64)):
        offs, vals = inputs.c2_input(dt, nseg=1 << 12)
        assert digest(offs, vals) == dig[f"c2_{tag}_2^12seg"]["in"]
        a = vals.copy()
        for s in range(len(offs) - 1):
            lo, hi = int(offs[s]), int(offs[s + 1])
            oracle.smallsort_region(a, lo, hi - lo, oracle.sentinel_for(a))
        assert digest(a) == dig[f"c2_{tag}_2^12seg"]["out"]
    x = inputs.c3_input(n=1 << 20)
    d = dig["c3_f64_2^20"]
    assert digest(x) == d["in"]
    pivot = x[oracle.median3_index(x, 0, len(x) - 1)]
    assert float(pivot) == d["pivot"]
    a = x.copy()
    b = oracle.partition_region(a, pivot)
    assert b == d["split"] and digest(a) == d["layout"]
    k0, v0 = inputs.c4_input(n=1 << 18)
    d = dig["c4_kv_2^18"]
    assert digest(k0, v0) == d["in"]
    k, v = k0.copy(), v0.copy()
    oracle.kv_sort(k, v)
    assert digest(k) == d["keys"] and digest(v) == d["vals"]
    for dist in ("uniform", "sorted", "reverse", "few"):
        for tag, dt in (("i32", np.int32), ("f64", np.float64)):
            x = inputs.c5_input(dt, dist, n=1 << 16)
            d = dig[f"c5_{tag}_{dist}_2^16"]
            assert digest(x) == d["in"]
            a = x.copy()
            oracle.sort(a)
            assert digest(a) == d["out"]


def test_sort_bound_validation():
    a = np.zeros(10, dtype=np.float64)
    with pytest.raises(AssertionError):
        oracle.quicksort(a, 8, 129, np.inf)  # bound > 16*L (quicksort.py:51)


def test_c5_chunking_independent_of_rank_count():
    for dist in ("uniform", "few", "reverse"):
        whole = inputs.c5_input(np.int32, dist, n=1 << 12)
        parts = [inputs.c5_input(np.int32, dist, n=1 << 12, rank=r, world=4) for r in range(4)]
        assert np.array_equal(whole, np.concatenate(parts))
