"""Drop-in proof through the reference's own callers.

integration/_kernels_b200.py replaces the reference's native kernel module
``vexsort._kernels`` with ctypes bindings of the B200 C ABI.  These tests
run the REFERENCE package (its copy in baseline/_ref, made by
tests/golden/make_golden.py) with that module installed, so every call the
reference's API makes at quicksort.py:124-133, partition.py:134-145,
smallsort.py:235-239 and keyvalue.py:90-94/150-161/240-249 lands in the B200
kernels:

* every NATIVE-backend case of the reference's own test files
  (test_quicksort.py, test_smallsort.py, test_partition.py: the cases that
  reach ``_kernels``) -- minus the one that pins the CPU partition's exact
  LAYOUT (a documented deviation: the boundary and both sides as multisets
  are identical, the order inside a side is not).  The emulated-backend
  cases are pure-Python models of the CPU lanes (minutes of CPU each) and
  never call ``_kernels``;
* the reference's kv_sort / kv_partition_region on C4-style inputs, which
  the reference itself only checks in its bench gate.
"""

from __future__ import annotations

import os
import subprocess
import sys
import textwrap

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
LAYOUT_TESTS = ["test_partition_backends_bit_identical", "test_scalar_partition_contract"]


def _need_ref():
    if not (os.path.isdir(os.path.join(REF, "vexsort")) and os.path.isdir(os.path.join(REF, "tests"))):
        pytest.skip("reference copy missing (run tests/golden/make_golden.py in the authoring container)")


def _env():
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, ROOT, env.get("PYTHONPATH", "")])
    env["NUMBA_CACHE_DIR"] = "/tmp/numba_cache_ref"
    return env


def test_reference_test_suite_through_b200_kernels():
    _need_ref()
    tests = [os.path.join(REF, "tests", f) for f in ("test_quicksort.py", "test_smallsort.py", "test_partition.py")]
    sel = "native and " + " and ".join(f"not {t}" for t in LAYOUT_TESTS)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "integration.ref_plugin", "-k", sel,
                        "-p", "no:cacheprovider", "--timeout", "240", *tests], cwd=REF, env=_env(),
                       capture_output=True, text=True, timeout=900)
    tail = (r.stdout + r.stderr)[-3000:]
    assert r.returncode == 0, tail
    assert "_kernels_b200 calls:" in tail and "'quicksort'" in tail and "'partition'" in tail, tail
    assert " passed" in tail and "failed" not in tail, tail


def test_reference_kv_api_through_b200_kernels():
    _need_ref()
    code = textwrap.dedent("""
        import numpy as np
        import integration._kernels_b200 as kb
        kb.install()
        import vexsort
        from vexsort.quicksort import SortConfig
        rng = np.random.default_rng(4)
        for n in (0, 1, 300, 5000, 1 << 18, 1 << 21):
            k = rng.integers(0, 2**31, size=n, dtype=np.int32)
            v = np.arange(n, dtype=np.int32)
            k0 = k.copy()
            vexsort.kv_sort(k, v)
            assert np.array_equal(k, np.sort(k0)) and np.array_equal(k0[v], k)
            assert np.array_equal(np.sort(v), np.arange(n))
            kf = rng.uniform(-1e6, 1e6, size=n)
            vf = np.arange(n, dtype=np.int64)
            kf0 = kf.copy()
            vexsort.kv_sort(kf, vf, SortConfig(pivot_strategy="random", pivot_seed=3))
            assert np.array_equal(kf, np.sort(kf0)) and np.array_equal(kf0[vf], kf)
            k = k0.copy(); v = np.arange(n, dtype=np.int32)
            p = int(rng.integers(0, 2**31))
            b = vexsort.kv_partition_region(k, v, p)
            assert b == int((k0 <= p).sum()) and np.all(k[:b] <= p) and np.all(k[b:] > p)
            assert np.array_equal(k0[v], k)
        x = rng.integers(-2**31, 2**31 - 1, size=1 << 22, dtype=np.int32, endpoint=True)
        y = x.copy()
        vexsort.sort(y)
        assert np.array_equal(y, np.sort(x))
        assert kb.CALLS.get("kv_quicksort", 0) >= 8 and kb.CALLS.get("quicksort", 0) >= 1, kb.CALLS
        print("ok", kb.CALLS)
    """)
    r = subprocess.run([sys.executable, "-c", code], cwd=REF, env=_env(), capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0 and "ok" in r.stdout, (r.stdout + r.stderr)[-3000:]


def test_stub_quicksort_many_pipelined():
    """The stub's pipelined loop (vx_host_sort_submit / vx_host_sort_wait)
    gives what one `_kernels.quicksort` call per array gives."""
    import numpy as np

    sys.path.insert(0, ROOT)
    import integration._kernels_b200 as kb

    rng = np.random.default_rng(2)
    arrays = [rng.integers(-(2**31), 2**31 - 1, size=n, dtype=np.int32) for n in (5, 70000, 1 << 20, 0, 333, 1 << 19)]
    arrays += [rng.standard_normal(n) for n in (1, 4097, 1 << 18)]
    want = [np.sort(a) for a in arrays]
    kb.quicksort_many([a for a in arrays if a.dtype == np.int32], 16, 256, 2**31 - 1, 0, False, False, 0)
    kb.quicksort_many([a for a in arrays if a.dtype == np.float64], 8, 128, np.inf, 0, False, False, 0)
    for a, w in zip(arrays, want):
        assert np.array_equal(a, w)
    assert kb.CALLS.get("quicksort_many") == 2
