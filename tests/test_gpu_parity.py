"""GPU parity: the B200 kernels (through the C ABI) against the CPU oracle
and the reference-generated golden fixtures.

Rules: int32 / float64 sorts bit-exact; partitions: exact
boundary, side predicates, multiset (the reference's layout is a CPU
artefact); kv: keys bit-exact, keys_in[vals_out] == keys_out and vals_out a
permutation (pair-multiset equality).
"""

import json
import os

import numpy as np
import pytest

import inputs
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1704_08579_b200 as vx  # noqa: E402

DEV = "cuda"


def _d(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def _h(t):
    return t.cpu().numpy()


def _load(golden_dir, name):
    return np.load(os.path.join(golden_dir, name))


def _ids(z):
    return sorted({k.rsplit("_", 1)[0] for k in z.files})


def _digests(golden_dir):
    with open(os.path.join(golden_dir, "config_digests.json")) as f:
        return json.load(f)


def _digest(*arrs):
    from make_golden import digest

    return digest(*arrs)


# ------------------------------------------------------------------ sort


def test_reference_example():
    for dt in (np.int32, np.float64):
        t = _d(np.array([3, 1, 2, 0, 5], dtype=dt))
        vx.sort(t)
        assert _h(t).tolist() == [0, 1, 2, 3, 5]


def test_trivial_regions():
    for dt in (np.int32, np.float64):
        for data in ([], [4], [7, 7, 7, 7]):
            t = _d(np.array(data, dtype=dt))
            vx.sort(t)
            assert _h(t).tolist() == sorted(data)


def test_golden_sort_cases_device(golden_dir):
    z = _load(golden_dir, "sort_cases.npz")
    for cid in _ids(z):
        x, want = z[cid + "_in"], z[cid + "_out"]
        for strategy in ("median3", "middle", "random"):
            t = _d(x)
            vx.sort(t, vx.SortConfig(pivot_strategy=strategy, pivot_seed=9))
            assert np.array_equal(_h(t), want), (cid, strategy)


def test_golden_sort_cases_host_buffers(golden_dir):
    # numpy arrays in, in place, through the host-buffer C ABI (vx_host_*)
    z = _load(golden_dir, "sort_cases.npz")
    for cid in _ids(z):
        x, want = z[cid + "_in"], z[cid + "_out"]
        a = x.copy()
        vx.sort(a)
        assert np.array_equal(a, want), cid


@pytest.mark.parametrize("dt", [np.int32, np.float64])
def test_random_sizes_match_oracle(dt):
    rng = np.random.default_rng(1)
    sizes = rng.integers(0, 70000, size=30).tolist() + [0, 1, 2, 255, 256, 257, 4095, 4096, 4097, 8191, 8192,
                                                       8193, 16385, 100003]
    for n in sizes:
        x = (rng.integers(-(2**31), 2**31 - 1, size=n, dtype=np.int64, endpoint=True).astype(np.int32)
             if dt == np.int32 else rng.uniform(-1e9, 1e9, size=n))
        t = _d(x)
        vx.sort(t)
        want = x.copy()
        oracle.sort(want)
        assert np.array_equal(_h(t), want), n


@pytest.mark.parametrize("dt", [np.int32, np.float64])
@pytest.mark.parametrize("n", [1 << 16, 1 << 20])
def test_adversarial_patterns(dt, n):
    pats = {
        "sorted": np.arange(n),
        "reverse": np.arange(n)[::-1].copy(),
        "sawtooth": np.tile(np.arange(37), n // 37 + 1)[:n],
        "few-distinct": np.random.default_rng(5).integers(0, 8, size=n),
        "all-equal": np.full(n, 7),
        "two-values": np.random.default_rng(6).integers(0, 2, size=n) * 1000,
        "organ-pipe": np.concatenate([np.arange(n // 2), np.arange(n - n // 2)[::-1]]),
    }
    for name, base in pats.items():
        x = base.astype(dt)
        t = _d(x)
        vx.sort(t)
        assert np.array_equal(_h(t), np.sort(x)), name


@pytest.mark.parametrize("dt", [np.int32, np.float64])
def test_extreme_values_and_sentinels(dt):
    rng = np.random.default_rng(77)
    for n in (100, 300, 5000, 50000, 300000):
        x = rng.integers(-50, 50, size=n).astype(dt)
        if dt == np.int32:
            x[::7] = np.iinfo(np.int32).max
            x[3::11] = np.iinfo(np.int32).min
        else:
            x[::7] = np.inf
            x[3::11] = -np.inf
            x[5::13] = np.finfo(np.float64).max
        t = _d(x)
        vx.sort(t)
        assert np.array_equal(_h(t), np.sort(x)), n


def test_custom_sort_bound_and_flags():
    rng = np.random.default_rng(3)
    for dt, lanes in ((np.int32, 16), (np.float64, 8)):
        x = rng.integers(-100, 100, size=40000).astype(dt)
        for cfg in (vx.SortConfig(sort_bound=lanes), vx.SortConfig(sort_bound=1),
                    vx.SortConfig(skip_empty_stores=True, swap_buffered=True)):
            t = _d(x)
            vx.sort(t, cfg)
            assert np.array_equal(_h(t), np.sort(x))


def test_sort_bound_validation():
    with pytest.raises(AssertionError):
        vx.sort(_d(np.zeros(300, dtype=np.float64)), vx.SortConfig(sort_bound=129))
    with pytest.raises(ValueError):
        vx.SortConfig(pivot_strategy="bogus")


def test_sort_is_idempotent():
    x = np.random.default_rng(21).integers(-(2**31), 2**31 - 1, size=200000, dtype=np.int32)
    t = _d(x)
    vx.sort(t)
    once = _h(t).copy()
    vx.sort(t)
    assert np.array_equal(_h(t), once)


def test_sort_views_in_place():
    x = np.random.default_rng(2).integers(-1000, 1000, size=50000).astype(np.int32)
    t = _d(x)
    vx.sort(t[1000:40001])
    want = x.copy()
    want[1000:40001] = np.sort(want[1000:40001])
    assert np.array_equal(_h(t), want)


def test_c1_digest_matches_reference(golden_dir):
    d = _digests(golden_dir)["c1_i32_2^20"]
    x = inputs.c1_input()
    assert _digest(x) == d["in"]
    t = _d(x)
    vx.sort(t)
    assert _digest(_h(t)) == d["out"]


@pytest.mark.parametrize("dist", ["uniform", "sorted", "reverse", "few"])
def test_c5_reduced_digests_match_reference(golden_dir, dist):
    dig = _digests(golden_dir)
    for tag, dt in (("i32", np.int32), ("f64", np.float64)):
        x = inputs.c5_input(dt, dist, n=1 << 16)
        d = dig[f"c5_{tag}_{dist}_2^16"]
        assert _digest(x) == d["in"]
        t = _d(x)
        vx.sort(t)
        assert _digest(_h(t)) == d["out"]


@pytest.mark.parametrize("dt", [np.int32, np.float64])
def test_large_sort_2_24(dt):
    n = 1 << 24
    rng = np.random.default_rng(11)
    x = (rng.integers(-(2**31), 2**31 - 1, size=n, dtype=np.int32, endpoint=True) if dt == np.int32
         else rng.uniform(-1e6, 1e6, size=n))
    t = _d(x)
    vx.sort(t)
    assert np.array_equal(_h(t), np.sort(x))


def test_full_size_c5_distributions_properties():
    # size-independent properties at 2^26 (sortedness + checksum of the
    # multiset) for the four C5 distributions generated on the device
    import ctypes

    L = vx._lib.lib()
    n = 1 << 26
    for dist in (0, 1, 2, 3):
        t = torch.empty(n, dtype=torch.int32, device=DEV)
        L.vx_generate(0, dist, ctypes.c_void_p(t.data_ptr()), n, 1, 0, n,
                      ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        ref = torch.sort(t.to(torch.int64))[0]  # independent comparator (library sort, test only)
        vx.sort(t)
        assert torch.equal(t.to(torch.int64), ref), dist


@pytest.mark.parametrize("shape", ["lognormal", "clusters", "spikes", "two_values"])
@pytest.mark.parametrize("dt", [torch.int32, torch.float64])
def test_skewed_keys_through_the_cta_local_level(shape, dt):
    """2^25 keys (large enough for the CTA-local level) whose local ranges
    are far from uniform: interpolation buckets overflow and segments fall
    back to sampled pivots; outer segments have no parent bounds; a segment
    can hold one repeated key.  Checked against torch.sort as an
    independent comparator."""
    n = 1 << 25
    g = torch.Generator(device=DEV).manual_seed(7)
    if shape == "lognormal":
        x = torch.exp(torch.randn(n, device=DEV, generator=g, dtype=torch.float64) * 6.0)
    elif shape == "clusters":  # 64 tight clusters with wide gaps
        c = torch.randint(0, 64, (n,), device=DEV, generator=g).to(torch.float64)
        x = c * 1e7 + torch.randn(n, device=DEV, generator=g, dtype=torch.float64) * 50.0
    elif shape == "spikes":  # 90 % of the keys on 8 values, the rest uniform
        u = torch.rand(n, device=DEV, generator=g, dtype=torch.float64)
        spike = torch.randint(0, 8, (n,), device=DEV, generator=g).to(torch.float64) * 1e6
        x = torch.where(u < 0.9, spike, torch.rand(n, device=DEV, generator=g, dtype=torch.float64) * 8e6)
    else:  # two values, alternating blocks
        x = ((torch.arange(n, device=DEV) // 4096) % 2).to(torch.float64) * 3.0
    if dt == torch.int32:
        x = torch.clamp(x, -2.0e9, 2.0e9).to(torch.int32)
    t = x.to(dt).contiguous()
    ref = torch.sort(t.clone())[0]
    vx.sort(t)
    assert torch.equal(t, ref), (shape, dt)


# ------------------------------------------------------------- partition


def test_partition_example():
    for dt in (np.int32, np.float64):
        t = _d(np.array([3, 1, 2, 0, 5], dtype=dt))
        b = vx.partition_region(t, 2)
        assert b == 3
        a = _h(t)
        assert sorted(a[:3].tolist()) == [0, 1, 2] and sorted(a[3:].tolist()) == [3, 5]


def _check_partitioned(arr, before, pivot, b):
    assert 0 <= b <= len(arr)
    assert np.all(arr[:b] <= pivot)
    assert np.all(arr[b:] > pivot)
    assert np.array_equal(np.sort(arr), np.sort(before))
    assert b == int(np.count_nonzero(before <= pivot))


def test_golden_partition_cases(golden_dir):
    z = _load(golden_dir, "partition_cases.npz")
    for cid in _ids(z):
        x = z[cid + "_in"]
        b_want, opt_a, opt_b = (int(v) for v in z[cid + "_meta"])
        pivot = float(z[cid + "_pivot"][0])
        if x.dtype == np.int32:
            pivot = int(pivot)
        want = z[cid + "_out"]
        t = _d(x)
        b = vx.partition_region(t, pivot, skip_empty_stores=bool(opt_a), swap_buffered=bool(opt_b))
        assert b == b_want, cid
        got = _h(t)
        _check_partitioned(got, x, pivot, b)
        # same sides as the reference's own layout (as multisets)
        assert np.array_equal(np.sort(got[:b]), np.sort(want[:b]))
        assert np.array_equal(np.sort(got[b:]), np.sort(want[b:]))
        # host-buffer path too
        a = x.copy()
        assert vx.partition_region(a, pivot) == b_want
        _check_partitioned(a, x, pivot, b_want)


def test_partition_empty_tiny_all_low_all_high():
    for dt in (np.int32, np.float64):
        for n in (0, 1, 2, 5, 33, 4097):
            x = np.full(n, 3, dtype=dt)
            assert vx.partition_region(_d(x), 2) == 0
            assert vx.partition_region(_d(x), 3) == n  # ties go low
        rng = np.random.default_rng(0)
        x = rng.integers(-10, 10, size=100000).astype(dt)
        assert vx.partition_region(_d(x), 10) == 100000
        assert vx.partition_region(_d(x), -11) == 0


def test_partition_pivot_semantics_int32():
    x = np.arange(-10, 10, dtype=np.int32)
    assert vx.partition_region(_d(x), 2.5) == 13      # floor(2.5) = 2
    assert vx.partition_region(_d(x), -2.5) == 8      # floor(-2.5) = -3: -10..-3
    assert vx.partition_region(_d(x), 2**40) == 20
    assert vx.partition_region(_d(x), -(2**40)) == 0
    assert vx.partition_region(_d(x), float("nan")) == 0


@pytest.mark.parametrize("dt", [np.int32, np.float64])
def test_partition_random_sweep_vs_oracle(dt):
    rng = np.random.default_rng(42)
    for _ in range(60):
        n = int(rng.integers(0, 300000))
        x = rng.integers(-100, 100, size=n).astype(dt)
        pivot = int(rng.integers(-110, 110))
        t = _d(x)
        b = vx.partition_region(t, pivot)
        assert b == oracle.partition_region(x.copy(), pivot)
        _check_partitioned(_h(t), x, pivot, b)


def test_partition_misaligned_views_and_out():
    rng = np.random.default_rng(4)
    x = rng.standard_normal(100003)
    t = _d(x)
    v = t[3:]  # not 16-byte aligned -> scalar-load kernel variant
    out = torch.empty_like(v)
    b = vx.partition_region(v, 0.1, out=out)
    _check_partitioned(_h(out), x[3:], 0.1, b)
    assert np.array_equal(_h(t), x)  # out= leaves the input untouched


def test_c3_reduced_digest_matches_reference(golden_dir):
    d = _digests(golden_dir)["c3_f64_2^20"]
    x = inputs.c3_input(n=1 << 20)
    assert _digest(x) == d["in"]
    pivot = float(x[oracle.median3_index(x, 0, len(x) - 1)])
    assert pivot == d["pivot"]
    t = _d(x)
    b = vx.partition_region(t, pivot)
    assert b == d["split"]
    got = _h(t)
    assert _digest(np.sort(got[:b])) == d["sorted_low"]
    assert _digest(np.sort(got[b:])) == d["sorted_high"]


def test_c3_full_size_split_exact():
    # 2^28 f64 N(0,1) generated on device; split vs an independent count
    import ctypes

    n = 1 << 28
    L = vx._lib.lib()
    x = torch.empty(n, dtype=torch.float64, device=DEV)
    L.vx_generate(1, 4, ctypes.c_void_p(x.data_ptr()), n, 3, 0, n,
                  ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    pivot = float(x[vx.select_pivot(x, 0, n - 1)].item())
    out = torch.empty_like(x)
    b = vx.partition_region(x, pivot, out=out)
    assert b == int((x <= pivot).sum().item())
    assert bool((out[:b] <= pivot).all()) and bool((out[b:] > pivot).all())
    assert float(out.sum().item()) == pytest.approx(float(x.sum().item()), rel=1e-9, abs=1e-6)
    assert torch.equal(torch.sort(out[:b])[0], torch.sort(x[x <= pivot])[0])


# -------------------------------------------------------------- small sort


def test_golden_smallsort_all_lengths(golden_dir):
    z = _load(golden_dir, "smallsort_cases.npz")
    for cid in _ids(z):
        x, want = z[cid + "_in"], z[cid + "_out"]
        t = _d(x)
        vx.sort_small_region(t)
        assert np.array_equal(_h(t), want), cid


def test_smallsort_rejects_oversize():
    with pytest.raises(AssertionError):
        vx.sort_small_region(_d(np.zeros(257, dtype=np.int32)))
    with pytest.raises(AssertionError):
        vx.sort_small_region(_d(np.zeros(129, dtype=np.float64)))


def test_padding_value_never_leaks():
    for dt, sent in ((np.int32, 2**31 - 1), (np.float64, np.inf)):
        for n in (1, 7, 19, 128):
            t = _d(np.full(n, sent, dtype=dt))
            vx.sort_small_region(t)
            assert np.all(_h(t) == sent)


@pytest.mark.parametrize("tag,dt", [("i32", np.int32), ("f64", np.float64)])
def test_c2_reduced_digest_matches_reference(golden_dir, tag, dt):
    d = _digests(golden_dir)[f"c2_{tag}_2^12seg"]
    offs, vals = inputs.c2_input(dt, nseg=1 << 12)
    assert _digest(offs, vals) == d["in"]
    t = _d(vals)
    vx.sort_segments(t, _d(offs))
    assert _digest(_h(t)) == d["out"]


def test_segments_every_length_and_payload():
    rng = np.random.default_rng(9)
    lens = np.concatenate([np.arange(0, 257), rng.integers(0, 257, size=3000)])
    offs = np.zeros(len(lens) + 1, dtype=np.int64)
    np.cumsum(lens, out=offs[1:])
    for dt, vdt in ((np.int32, np.int32), (np.float64, np.int64)):
        k = rng.integers(-20, 20, size=int(offs[-1])).astype(dt)
        v = np.arange(len(k), dtype=vdt)
        tk, tv = _d(k), _d(v)
        vx.sort_segments(tk, _d(offs), tv)
        gk, gv = _h(tk), _h(tv)
        for s in range(len(lens)):
            lo, hi = offs[s], offs[s + 1]
            assert np.array_equal(gk[lo:hi], np.sort(k[lo:hi]))
            assert np.array_equal(np.sort(gv[lo:hi]), v[lo:hi])
        assert np.array_equal(k[gv], gk)


def test_segments_reject_long():
    offs = np.array([0, 10, 300], dtype=np.int64)
    with pytest.raises(AssertionError):
        vx.sort_segments(_d(np.zeros(300, dtype=np.int32)), _d(offs))


# ---------------------------------------------------------------------- kv


def _check_kv(k_in, k_out, v_out):
    assert np.array_equal(k_out, np.sort(k_in))
    assert np.array_equal(k_in[v_out], k_out)
    assert np.array_equal(np.sort(v_out), np.arange(len(k_in)))


def test_golden_kv_cases(golden_dir):
    z = _load(golden_dir, "kv_cases.npz")
    for tag, vdt in (("i32", np.int32), ("f64", np.int64)):
        for i in range(80):
            key = f"sort_{tag}_{i}"
            if key + "_kin" not in z.files:
                continue
            kin = z[key + "_kin"]
            tk, tv = _d(kin), _d(np.arange(len(kin), dtype=vdt))
            vx.kv_sort(tk, tv)
            assert np.array_equal(_h(tk), z[key + "_kout"])
            _check_kv(kin, _h(tk), _h(tv))
            # kv partition: boundary exact, sides as multisets of pairs
            pk = f"part_{tag}_{i}"
            b_want, pivot = (int(t) for t in z[pk + "_meta"])
            tk, tv = _d(kin), _d(np.arange(len(kin), dtype=vdt))
            b = vx.kv_partition_region(tk, tv, pivot)
            assert b == b_want
            gk, gv = _h(tk), _h(tv)
            assert np.array_equal(kin[gv], gk)
            assert np.all(gk[:b] <= pivot) and np.all(gk[b:] > pivot)
            assert np.array_equal(np.sort(gv[:b]), np.sort(z[pk + "_vout"][:b]))


def test_kv_host_buffers_and_alias():
    rng = np.random.default_rng(5)
    k = rng.integers(0, 50, size=20000).astype(np.int32)
    v = np.arange(len(k), dtype=np.int32)
    k2, v2 = k.copy(), v.copy()
    vx.sort_kv(k2, v2)
    _check_kv(k, k2, v2)


def test_kv_width_rule():
    with pytest.raises(AssertionError):
        vx.kv_sort(_d(np.zeros(10, dtype=np.int32)), _d(np.zeros(10, dtype=np.int64)))
    with pytest.raises(AssertionError):
        vx.kv_sort(_d(np.zeros(10, dtype=np.int32)), _d(np.zeros(11, dtype=np.int32)))


@pytest.mark.parametrize("kdt,vdt", [(np.int32, np.float32), (np.int32, np.uint32), (np.float64, np.float64),
                                     (np.float64, np.int64)])
def test_kv_value_dtypes_move_as_raw_bits(kdt, vdt):
    """any same-width value type (keyvalue.py:44-47) rides
    along bit for bit; sizes cover the finish and the CTA-local level."""
    rng = np.random.default_rng(11)
    for n in (3000, 1 << 20):
        k = rng.integers(-5000, 5000, size=n).astype(kdt)
        idx = np.arange(n)
        v = (idx * 2.5).astype(vdt) if np.dtype(vdt).kind == "f" else idx.astype(vdt)
        tk, tv = _d(k), _d(v)
        vx.kv_sort(tk, tv)
        gk, gv = _h(tk), _h(tv)
        assert np.array_equal(gk, np.sort(k))
        orig = (gv / 2.5).astype(np.int64) if np.dtype(vdt).kind == "f" else gv.astype(np.int64)
        assert np.array_equal(np.sort(orig), idx)  # a permutation of the payloads
        assert np.array_equal(k[orig], gk)  # every payload still sits next to its key


def test_c4_reduced_digest_and_pairs(golden_dir):
    d = _digests(golden_dir)["c4_kv_2^18"]
    k0, v0 = inputs.c4_input(n=1 << 18)
    assert _digest(k0, v0) == d["in"]
    tk, tv = _d(k0), _d(v0)
    vx.kv_sort(tk, tv)
    assert _digest(_h(tk)) == d["keys"]
    _check_kv(k0, _h(tk), _h(tv))


def test_kv_f64_large():
    rng = np.random.default_rng(8)
    n = 1 << 22
    k = rng.integers(-1000, 1000, size=n).astype(np.float64)
    tk, tv = _d(k), _d(np.arange(n, dtype=np.int64))
    vx.kv_sort(tk, tv)
    _check_kv(k, _h(tk), _h(tv))


def test_c4_full_size_properties():
    # 2^28 pairs: keys sorted (vs library sort as an independent comparator),
    # values a permutation with keys_in[vals_out] == keys_out
    import ctypes

    n = 1 << 28
    L = vx._lib.lib()
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    k = torch.empty(n, dtype=torch.int32, device=DEV)
    v = torch.empty(n, dtype=torch.int32, device=DEV)
    L.vx_generate(0, 5, ctypes.c_void_p(k.data_ptr()), n, 4, 0, n, st)
    L.vx_generate(0, 6, ctypes.c_void_p(v.data_ptr()), n, 4, 0, n, st)
    k0 = k.clone()
    vx.kv_sort(k, v)
    assert torch.equal(k, torch.sort(k0)[0])
    assert torch.equal(k0[v.long()], k)
    assert bool((torch.bincount(v.long(), minlength=n) == 1).all())


# ---------------------------------------------------------- sharded (P=1)


def test_sharded_single_rank_and_bucket_partition():
    import torch.distributed as dist

    assert not dist.is_initialized()
    rng = np.random.default_rng(12)
    x = rng.integers(0, 16, size=300000).astype(np.int32)
    out = vx.sharded_sort(_d(x))
    assert np.array_equal(_h(out), np.sort(x))
    # bucket partition with (key, index) splitters against a numpy model
    from paper_1704_08579_b200.sharded import B200Ops

    ops = B200Ops()
    gofs = 12345
    pos = np.sort(rng.choice(len(x), size=4000, replace=False))
    sk, si = ops.select_splitters(_d(x[pos]), _d(pos + gofs), 8)
    order = np.lexsort((pos + gofs, x[pos]))
    q = [(r * 4000) // 8 for r in range(1, 8)]
    assert np.array_equal(_h(sk), x[pos][order][q]) and np.array_equal(_h(si), (pos + gofs)[order][q])
    parted, counts = ops.bucket_partition(_d(x), gofs, sk, si)
    gk, gi = _h(sk), _h(si)
    gidx = np.arange(len(x)) + gofs
    dest = np.zeros(len(x), dtype=np.int64)
    for j in range(len(gk)):
        dest += (gk[j] < x) | ((gk[j] == x) & (gi[j] < gidx))
    want_counts = np.bincount(dest, minlength=8)
    assert np.array_equal(_h(counts), want_counts)
    p = _h(parted)
    o = 0
    for b in range(8):
        assert np.array_equal(np.sort(p[o:o + want_counts[b]]), np.sort(x[dest == b]))
        o += want_counts[b]


# ------------------------------------------------------ extra device APIs


@pytest.mark.parametrize("dt", [np.int32, np.float64])
def test_sort_into_leaves_input_untouched(dt):
    rng = np.random.default_rng(31)
    for n in (0, 1, 5, 300, 9000, 1 << 20):
        x = (rng.integers(-(2**31), 2**31 - 1, size=n, dtype=np.int64, endpoint=True).astype(np.int32)
             if dt == np.int32 else rng.uniform(-1e6, 1e6, size=n))
        src = _d(x)
        out = torch.empty_like(src)
        vx.sort_into(src, out)
        assert np.array_equal(_h(out), np.sort(x))
        assert np.array_equal(_h(src), x)


def test_kv_sort_into_f64_pairs():
    rng = np.random.default_rng(32)
    n = 300000
    k = rng.integers(-500, 500, size=n).astype(np.float64)
    v = np.arange(n, dtype=np.int64)
    tk, tv = _d(k), _d(v)
    ok, ov = torch.empty_like(tk), torch.empty_like(tv)
    vx.sort_into(tk, ok, values=tv, out_values=ov)
    _check_kv(k, _h(ok), _h(ov))
    assert np.array_equal(_h(tk), k) and np.array_equal(_h(tv), v)


def test_kv_partition_f64_out_of_place():
    rng = np.random.default_rng(33)
    n = 200003
    k = rng.standard_normal(n)
    v = np.arange(n, dtype=np.int64)
    tk, tv = _d(k), _d(v)
    ok, ov = torch.empty_like(tk), torch.empty_like(tv)
    b = vx.kv_partition_region(tk, tv, 0.25, out=(ok, ov))
    gk, gv = _h(ok), _h(ov)
    assert b == int(np.count_nonzero(k <= 0.25))
    assert np.all(gk[:b] <= 0.25) and np.all(gk[b:] > 0.25)
    assert np.array_equal(k[gv], gk) and np.array_equal(np.sort(gv), v)


def test_profile_counters_report_launches_and_elements():
    import ctypes

    L = vx._lib.lib()
    L.vx_profile_reset()
    L.vx_profile_enable(1)
    n = 1 << 24  # large enough for the CTA-local level (256 target-sized segments)
    x = _d(np.random.default_rng(34).integers(-(2**31), 2**31 - 1, size=n, dtype=np.int32))
    vx.sort(x)
    torch.cuda.synchronize()
    L.vx_profile_enable(0)
    la = (ctypes.c_int64 * 9)()
    ms = (ctypes.c_double * 9)()
    el = (ctypes.c_uint64 * 9)()
    assert L.vx_profile_read(la, ms, el, 9) == 9
    assert la[3] >= 1 and la[4] >= 1 and la[8] >= 1  # scatter, finish, CTA-local level
    assert el[3] >= n  # the first level moves every element
    # every element ends in a finish item or a CTA-local segment, except the
    # few buckets that hold a single key (final as they are)
    assert n - n // 1000 <= el[4] + el[8] <= n
    assert el[8] >= n // 2  # uniform keys: most segments go through the CTA-local level
    assert ms[8] > 0.0


@pytest.mark.parametrize("dist", [1, 2, 3])
def test_c5_f64_distributions_2_24(dist):
    import ctypes

    n = 1 << 24
    L = vx._lib.lib()
    t = torch.empty(n, dtype=torch.float64, device=DEV)
    L.vx_generate(1, dist, ctypes.c_void_p(t.data_ptr()), n, 1, 0, n,
                  ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    ref = torch.sort(t)[0]  # independent comparator (library sort, test only)
    out = vx.sharded_sort(t)  # P = 1 path (out of place)
    assert torch.equal(out, ref)


# ------------------------------------------------- pipelined host sorts


@pytest.mark.parametrize("dt", [np.int32, np.float64])
def test_sort_many_pipelined_host_regions(dt):
    """sort_many == sort on every region (quicksort.py:137-143 per array),
    with pinned, pageable, empty and single-element regions in one stream."""
    rng = np.random.default_rng(11)
    sizes = [0, 1, 2, 257, 5000, 1 << 16, (1 << 20) + 3, 1 << 21, 77, 1 << 18]
    arrs = []
    for i, n in enumerate(sizes):
        a = (rng.integers(-(2**31), 2**31 - 1, size=n, endpoint=True).astype(np.int32) if dt is np.int32
             else rng.standard_normal(n) * 1e3)
        arrs.append(a)
    want = []
    for a in arrs:
        w = a.copy()
        oracle.sort(w)
        want.append(w)
    regs = [torch.from_numpy(a.copy()).pin_memory() if i % 2 == 0 else a.copy() for i, a in enumerate(arrs)]
    vx.sort_many(regs)
    for r, w in zip(regs, want):
        got = r.numpy() if isinstance(r, torch.Tensor) else r
        assert np.array_equal(got, w)
    # out-of-place: sources untouched, sorted copies in `out`
    srcs = [torch.from_numpy(a.copy()).pin_memory() for a in arrs]
    outs = [torch.empty_like(s).pin_memory() for s in srcs]
    vx.sort_many(srcs, out=outs)
    for s, a, o, w in zip(srcs, arrs, outs, want):
        assert np.array_equal(s.numpy(), a) and np.array_equal(o.numpy(), w)


def test_host_submit_wait_contract():
    """Tickets name one of two slots; a third submit waits for the oldest
    sort; the synchronous host calls may be mixed in; bad arguments fail the
    way the synchronous twins do."""
    import ctypes

    from paper_1704_08579_b200 import _lib

    L = _lib.lib()
    rng = np.random.default_rng(5)
    bufs = [torch.from_numpy(rng.integers(-1000, 1000, size=300000).astype(np.int32)).pin_memory() for _ in range(5)]
    want = [np.sort(b.numpy()) for b in bufs]
    tickets = []
    for b in bufs:
        t = ctypes.c_int(-1)
        p = ctypes.c_void_p(b.data_ptr())
        assert L.vx_host_sort_submit(0, p, None, p, None, b.numel(), 16, 0, 0, 0, ctypes.byref(t)) == 0
        assert t.value in (0, 1)
        tickets.append(t.value)
    x = rng.integers(-5, 5, size=1000).astype(np.int32)
    vx.sort(x)  # synchronous call while two submits are in flight
    assert np.array_equal(x, np.sort(x))
    assert L.vx_host_sort_wait(0) == 0 and L.vx_host_sort_wait(1) == 0
    assert L.vx_host_sort_wait(0) == 0  # idempotent
    for b, w in zip(bufs, want):
        assert np.array_equal(b.numpy(), w)
    assert L.vx_host_sort_wait(7) == -1
    t = ctypes.c_int(-1)
    p = ctypes.c_void_p(bufs[0].data_ptr())
    assert L.vx_host_sort_submit(0, p, None, p, None, 10, 8, 0, 0, 0, ctypes.byref(t)) == -1  # lane / kind mismatch
    assert L.vx_host_sort_submit(5, p, None, p, None, 10, 16, 0, 0, 0, ctypes.byref(t)) == -2  # dtype
    assert L.vx_host_sort_submit(0, p, p, p, None, 10, 16, 0, 0, 0, ctypes.byref(t)) == -1  # values: both or neither
    L.vx_host_release()


def test_host_submit_wait_pairs_out_of_place():
    """Pipelined key/value sorts (vx_host_sort_submit with values): keys
    bit-exact, values still name their keys, sources untouched."""
    import ctypes

    from paper_1704_08579_b200 import _lib

    L = _lib.lib()
    rng = np.random.default_rng(9)
    vp = ctypes.c_void_p
    jobs = []
    for n, kdt, vdt, lane in ((200000, np.int32, np.int32, 16), (1 << 20, np.float64, np.int64, 8),
                              (4099, np.int32, np.int32, 16)):
        k = (rng.integers(0, 2**31, size=n).astype(kdt) if kdt is np.int32 else rng.standard_normal(n))
        v = np.arange(n, dtype=vdt)
        sk, sv = torch.from_numpy(k.copy()).pin_memory(), torch.from_numpy(v.copy()).pin_memory()
        dk, dv = torch.empty_like(sk).pin_memory(), torch.empty_like(sv).pin_memory()
        t = ctypes.c_int(-1)
        rc = L.vx_host_sort_submit(0 if kdt is np.int32 else 1, vp(sk.data_ptr()), vp(sv.data_ptr()),
                                   vp(dk.data_ptr()), vp(dv.data_ptr()), n, lane, 0, 0, 0, ctypes.byref(t))
        assert rc == 0, L.vx_last_error()
        jobs.append((k, v, sk, sv, dk, dv, t.value))
    for k, v, sk, sv, dk, dv, t in jobs:
        assert L.vx_host_sort_wait(t) == 0
        assert np.array_equal(sk.numpy(), k) and np.array_equal(sv.numpy(), v)
        assert np.array_equal(dk.numpy(), np.sort(k))
        assert np.array_equal(k[dv.numpy()], dk.numpy())
        assert np.array_equal(np.sort(dv.numpy()), v)
    L.vx_host_release()


# ------------------------------------------- monotone inputs (presort.cuh)


def _stats_sort_into(src, **kw):
    out = torch.empty_like(src)
    st = {}
    vx.sort_into(src, out, stats=st, **kw)
    return out, st


@pytest.mark.parametrize("dt", [np.int32, np.float64])
def test_monotone_inputs_leave_before_level_0(dt):
    """Sorted and reverse-sorted inputs from 2^24 keys are recognised (one
    read pass) and copied / reversed instead of partitioned; the output is
    np.sort's either way, in place and out of place."""
    n = (1 << 24) + 77
    base = np.sort(inputs.c5_input(dt, "uniform", n=1 << 25)[:n])
    for name, x in (("sorted", base), ("reverse", base[::-1].copy()), ("equal", np.full(n, 7, dtype=dt))):
        t = _d(x)
        out, st = _stats_sort_into(t)
        assert st["scatter_elems"] == 0 and st["local_elems"] == 0 and st["finish_elems"] == n, (name, st)
        assert torch.equal(t, _d(x)), "input of an out-of-place sort was modified"
        assert np.array_equal(_h(out), base if name != "equal" else x), name
        vx.sort(t)  # in place
        assert np.array_equal(_h(t), base if name != "equal" else x), name


def test_almost_monotone_inputs_still_sort():
    """One inversion anywhere -- first pair, last pair, a CTA chunk boundary,
    between the sampled pairs -- sends the sort down the normal path."""
    n = 1 << 24
    base = np.sort(inputs.c5_input(np.int32, "uniform", n=n))
    rng = np.random.default_rng(8)
    spots = [0, n - 2, n // 2, (n - 1) // 592, 12345677] + rng.integers(0, n - 1, size=3).tolist()
    for rev in (False, True):
        for p in spots:
            x = base[::-1].copy() if rev else base.copy()
            if x[p] == x[p + 1]:
                continue
            x[p], x[p + 1] = x[p + 1], x[p]
            out, st = _stats_sort_into(_d(x))
            assert st["scatter_elems"] > 0, (rev, p)
            assert np.array_equal(_h(out), base), (rev, p)


def test_monotone_pairs_and_plateaus():
    """Key/value sorts: non-decreasing keys keep their pairs where they are,
    non-increasing keys (plateaus of equal keys included) are reversed with
    their values."""
    n = 1 << 24
    k = np.sort(np.random.default_rng(4).integers(0, 1 << 20, size=n).astype(np.int32))
    v = np.arange(n, dtype=np.int32)
    for keys in (k, k[::-1].copy()):
        tk, tv = _d(keys), _d(v)
        ok, ov = torch.empty_like(tk), torch.empty_like(tv)
        st = {}
        vx.sort_into(tk, ok, values=tv, out_values=ov, stats=st)
        assert st["scatter_elems"] == 0, st
        gk, gv = _h(ok), _h(ov)
        assert np.array_equal(gk, k) and np.array_equal(keys[gv], gk)
        assert np.array_equal(np.sort(gv), v)
        vx.kv_sort(tk, tv)
        assert np.array_equal(_h(tk), k) and np.array_equal(keys[_h(tv)], k)
    kf = np.sort(np.random.default_rng(5).standard_normal(n))[::-1].copy()
    vf = np.arange(n, dtype=np.int64)
    tk, tv = _d(kf), _d(vf)
    vx.kv_sort(tk, tv)
    assert np.array_equal(_h(tk), kf[::-1]) and np.array_equal(kf[_h(tv)], kf[::-1])


@pytest.mark.parametrize("dt", [np.int32, np.float64])
def test_few_unique_scatters_straight_into_the_output(dt):
    """Every level-0 bucket of a few-unique input is final (keys equal to a
    pivot): an out-of-place sort scatters them straight into the output --
    no copy home -- and an in-place sort still copies them back."""
    n = (1 << 23) + 5
    x = inputs.c5_input(dt, "few", n=1 << 24)[:n]
    want = np.sort(x)
    t = _d(x)
    out, st = _stats_sort_into(t)
    assert st["scatter_elems"] == n and st["finish_elems"] == 0 and st["levels"] == 1, st
    assert np.array_equal(_h(out), want) and torch.equal(t, _d(x))
    st2 = {}
    vx.sort_into(t, t, stats=st2)  # in place: level 0 parks the buckets in scratch
    assert st2["scatter_elems"] == n and st2["finish_elems"] == n, st2
    assert np.array_equal(_h(t), want)
    # pairs travel with their keys
    k = _d(x)
    v = torch.arange(n, dtype=torch.int32 if dt is np.int32 else torch.int64, device=DEV)
    ok, ov = torch.empty_like(k), torch.empty_like(v)
    vx.sort_into(k, ok, values=v, out_values=ov)
    assert np.array_equal(_h(ok), want) and np.array_equal(x[_h(ov)], want)
    assert np.array_equal(np.sort(_h(ov)), np.arange(n))


def test_uniform_looking_samples_with_structure_underneath():
    """Inputs whose coarse quantiles look uniform over the int32 range (so the
    root level takes equal-width buckets) but which are not uniform below
    that: a lattice of 4096 values, a heavy cluster, a narrow spike on a
    uniform floor.  Skewed children fall back to sampled pivots; the output is
    np.sort's."""
    rng = np.random.default_rng(12)
    n = (1 << 24) + 11
    full = rng.integers(-(2**31), 2**31 - 1, size=n, dtype=np.int64, endpoint=True)
    cases = {
        "lattice": (full >> 20) << 20,
        "cluster": np.where(rng.random(n) < 0.02, 123456789, full),
        "spike": np.where(rng.random(n) < 0.03, 1000 + rng.integers(0, 64, size=n), full),
        "pairs": (full >> 1) << 1,
    }
    for name, x in cases.items():
        x = x.astype(np.int32)
        out, st = _stats_sort_into(_d(x))
        assert np.array_equal(_h(out), np.sort(x)), name
        k = _d(x)
        v = torch.arange(n, dtype=torch.int32, device=DEV)
        vx.kv_sort(k, v)
        assert np.array_equal(_h(k), np.sort(x)) and np.array_equal(x[_h(v)], _h(k)), name


def test_uniform_looking_float64_with_outliers():
    """float64 keys whose sample looks uniform between its own extremes (the
    root level then cuts equal-width buckets in value space) with keys BEYOND
    those extremes -- a handful of huge outliers, infinities, both zeros --
    which saturate into the edge buckets; also a lattice and a normal
    distribution (which fails the test and keeps sampled pivots)."""
    rng = np.random.default_rng(21)
    n = (1 << 24) + 3
    u = rng.uniform(-1e6, 1e6, size=n)
    out_idx = rng.choice(n, size=64, replace=False)
    a = u.copy()
    a[out_idx[:16]] = 1e12 * rng.uniform(1, 2, size=16)
    a[out_idx[16:32]] = -1e12 * rng.uniform(1, 2, size=16)
    a[out_idx[32:36]] = np.inf
    a[out_idx[36:40]] = -np.inf
    a[out_idx[40:44]] = 0.0
    a[out_idx[44:48]] = -0.0
    cases = {"outliers": a, "lattice": np.round(u / 512.0) * 512.0, "normal": rng.standard_normal(n),
             "positive": rng.uniform(1e-300, 1e-290, size=n)}
    for name, x in cases.items():
        out, st = _stats_sort_into(_d(x))
        got, want = _h(out), np.sort(x)
        assert np.array_equal(got, want), name  # (+0.0 == -0.0 under array_equal; any order of the two is a sort)
        assert np.array_equal(np.sort(got.view(np.uint64)), np.sort(x.view(np.uint64))), name  # same bit patterns


def test_both_zeros_survive_every_network():
    """+0.0 and -0.0 compare equal but are different keys: every sort path
    (warp networks of the segment sort and the finish kernel, lane networks
    of the CTA-local level) must return the input's multiset of BIT PATTERNS.
    A cross-lane comparator that let the high lane take its partner on a tie
    duplicated one zero and lost the other."""
    rng = np.random.default_rng(33)
    for n in (64, 256, 5000, 1 << 16, (1 << 21) + 7, 1 << 24):
        for frac in (0.5, 0.02):
            x = rng.standard_normal(n)
            z = rng.random(n) < frac
            x[z] = np.where(rng.random(int(z.sum())) < 0.5, 0.0, -0.0)
            t = _d(x)
            vx.sort(t)
            got = _h(t)
            assert np.array_equal(got, np.sort(x))
            assert np.array_equal(np.sort(got.view(np.uint64)), np.sort(x.view(np.uint64))), (n, frac)
    # segments of every length, half zeros of either sign
    lens = rng.integers(1, 257, size=4000)
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    x = rng.standard_normal(int(offs[-1]))
    z = rng.random(len(x)) < 0.5
    x[z] = np.where(rng.random(int(z.sum())) < 0.5, 0.0, -0.0)
    t = _d(x)
    vx.sort_segments(t, _d(offs))
    got = _h(t)
    for s in range(len(lens)):
        a, b = offs[s], offs[s + 1]
        assert np.array_equal(got[a:b], np.sort(x[a:b]))
        assert np.array_equal(np.sort(got[a:b].view(np.uint64)), np.sort(x[a:b].view(np.uint64))), s
