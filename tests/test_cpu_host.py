"""CPU-only tests: the C-ABI library loads and exports every symbol the
header declares; host-side logic of the Python mirror (validation, dtype
rules, pivot conversion, config) behaves like the reference.  No kernel is
launched here."""

import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    with open(os.path.join(ROOT, "include", "vexsort_b200.h")) as f:
        src = f.read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(vx_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    import paper_1704_08579_b200._lib as L

    lib = L.lib()
    syms = _header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert lib.vx_version() == 1
    # the shared object really is sm_100a code
    out = os.popen(f"cuobjdump --list-elf {L.lib_path()} 2>/dev/null").read()
    if out:
        assert "sm_100a" in out


def test_header_is_c_compatible(tmp_path):
    src = tmp_path / "t.c"
    src.write_text('#include "vexsort_b200.h"\nint main(void){vx_sort_config c = {0}; (void)c; return vx_version() == 0;}\n')
    rc = os.system(f"/usr/bin/gcc -std=c99 -Wall -Werror -fsyntax-only -I{ROOT}/include {src}")
    assert rc == 0


def test_workspace_sizes_are_monotone():
    import paper_1704_08579_b200._lib as L

    lib = L.lib()
    prev = 0
    for n in (0, 1, 1000, 1 << 20, 1 << 28, 1 << 32):
        w = lib.vx_sort_workspace_bytes(0, 0, n)
        assert w >= prev
        prev = w
    # a scratch copy of the keys plus a 2-byte bucket id per element
    n = 1 << 28
    assert n * (4 + 2) <= lib.vx_sort_workspace_bytes(0, 0, n) <= n * 4 * 1.65
    assert lib.vx_sort_workspace_bytes(0, 1, n) >= 2 * n * 4
    assert lib.vx_sort_workspace_bytes(7, 0, n) == 0  # bad dtype


def test_rejects_unsupported_dtype():
    import paper_1704_08579_b200 as vx

    with pytest.raises(TypeError):
        vx.sort(np.zeros(10, dtype=np.int64))
    with pytest.raises(TypeError):
        vx.partition_region(np.zeros(10, dtype=np.float32), 0)
    import torch

    with pytest.raises(TypeError):
        vx.sort(torch.zeros(10, dtype=torch.int64))


def test_c_abi_rejects_bad_dtype_without_gpu():
    import paper_1704_08579_b200._lib as L

    lib = L.lib()
    rc = lib.vx_sort(5, None, None, 10, None, None, 0, None)
    assert rc == -2
    assert b"dtype" in lib.vx_last_error()
    with pytest.raises(TypeError):
        L.check(rc)


def test_config_validation():
    import paper_1704_08579_b200 as vx

    with pytest.raises(ValueError):
        vx.SortConfig(pivot_strategy="bogus")
    from paper_1704_08579_b200.quicksort import _resolve_bound

    assert _resolve_bound(vx.SortConfig(), 16) == 256
    assert _resolve_bound(vx.SortConfig(), 8) == 128
    with pytest.raises(AssertionError):
        _resolve_bound(vx.SortConfig(sort_bound=129), 8)
    with pytest.raises(ValueError):
        vx.get_backend("bogus", "i32")
    with pytest.raises(vx.BackendUnavailable):
        vx.get_backend("emulated", "i32")
    assert vx.get_backend("auto", "i32") is vx.get_backend("native", vx.I32)


def test_pivot_conversion_matches_numba_semantics():
    from paper_1704_08579_b200._region import pivot_for
    from paper_1704_08579_b200.lanes import F64, I32

    x = np.arange(-10, 10, dtype=np.int32)
    for p in (2, 2.5, -2.5, 0.0, -0.0, 9.99, -10.01, np.int64(3), np.float32(-1.5), 2**40, -(2**40),
              float("inf"), float("-inf")):
        c, short = pivot_for(I32, p)
        want = int(np.count_nonzero(x <= p))
        if short == "none":
            got = 0
        elif short == "all":
            got = len(x)
        else:
            got = int(np.count_nonzero(x <= c.value))
        assert got == want, p
    c, short = pivot_for(F64, 1.25)
    assert short is None and c.value == 1.25


def test_select_pivot_kats():
    # test_quicksort.py:28-49 of the reference
    import itertools

    import paper_1704_08579_b200 as vx

    for perm in itertools.permutations([10, 20, 30]):
        arr = np.array(perm, dtype=np.int32)
        assert arr[vx.select_pivot(arr, 0, 2, "median3")] == 20
    assert vx.select_pivot(np.array([1, 2, 3], dtype=np.int32), 0, 2, "median3") == 1
    arr = np.array([3, 1, 2, 0, 5], dtype=np.int32)
    assert vx.select_pivot(arr, 0, 4, "middle") == 2
    for state in (0, 1, 2**63, 12345):
        assert 10 <= vx.select_pivot(np.arange(100, dtype=np.int32), 10, 40, "random", state) <= 40


def test_backend_unavailable_without_gpu():
    import torch

    import paper_1704_08579_b200 as vx

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    assert not vx.native_available()
    assert vx.available_backends() == ()


def test_kv_contract_checks():
    import paper_1704_08579_b200 as vx

    with pytest.raises(AssertionError):
        vx.kv_sort(np.zeros(10, dtype=np.int32), np.zeros(10, dtype=np.int64))
    with pytest.raises(AssertionError):
        vx.kv_sort(np.zeros(10, dtype=np.int32), np.zeros(9, dtype=np.int32))
