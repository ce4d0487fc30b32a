"""Bench CLI: the reference's own caller of the
hot path, re-pointed at the B200 API.  Pinned to the reference itself:
tests/golden/benchcli_ref_checksums.csv is the checksum column of the
reference's `python -m vexsort.benchcli --max-exp 14 --reps 1 --backend
native` (tests/golden/make_benchcli_golden.sh)."""

import csv
import io
import os

import numpy as np
import pytest

from paper_1704_08579_b200 import benchcli as bc

GOLD = os.path.join(os.path.dirname(__file__), "golden", "benchcli_ref_checksums.csv")


def _golden():
    return {(r["experiment"], r["elem_type"], int(r["n"]), r["algorithm"]): r["checksum"]
            for r in csv.DictReader(open(GOLD))}


def _expected_checksum(exp, et, n):
    """The gate's checksum for one (experiment, type, n), from the seeded
    input and numpy alone (the reference oracle)."""
    cli_t = "kv" if et == "kv_i32" else et
    rng = bc._rng(1, exp, cli_t, n)
    data = bc.make_input(cli_t, n, rng)
    if cli_t == "kv":
        k, v = data
        if exp == "partition":
            pivot = k[int(rng.integers(0, n))]
            m = k <= pivot
            kk = np.concatenate([k[m], k[~m]])
            vv = np.concatenate([v[m], v[~m]])
            return bc.checksum_partitioned_pairs(kk, vv, int(m.sum()))
        o = np.argsort(k, kind="stable")
        return bc.checksum_pairs(k[o], v[o])
    if exp == "partition":
        pivot = data[int(rng.integers(0, n))]
        return bc.checksum_partitioned(data, int(np.count_nonzero(data <= pivot)))
    return bc.checksum_sorted(np.sort(data))


def test_inputs_and_checksums_match_reference():
    gold = _golden()
    seen = set()
    for (exp, et, n, alg), want in gold.items():
        if (exp, et, n) in seen:
            continue
        seen.add((exp, et, n))
        if exp == "smallsort" and n % 17 not in (0, 1):  # a spread of lengths keeps this fast
            continue
        assert _expected_checksum(exp, et, n) == want, (exp, et, n)
    assert len(seen) > 400


def test_csv_round_trip(tmp_path):
    recs = [bc.BenchRecord("fullsort", "i32", 4, "vexsort", 5, 1.5e-5, 1.5e-5 / 8, "ab" * 8),
            bc.BenchRecord("partition", "kv_i32", 2, "baseline_partition", 20, 3e-6, 1.5e-6, "cd" * 8),
            bc.BenchRecord("fullsort", "i32", 2, "baseline_sort", 5, 1e-6, 5e-7, "ef" * 8)]
    buf = io.StringIO()
    bc.emit_csv(recs, buf)
    lines = buf.getvalue().splitlines()
    assert lines[0] == "experiment,elem_type,n,algorithm,reps,mean_seconds,normalized,checksum"
    assert [ln.split(",")[2] for ln in lines[1:]] == ["2", "4", "2"]  # (experiment, type, n, algorithm) order
    p = tmp_path / "r.csv"
    p.write_text(buf.getvalue())
    back = bc.load_records(str(p))
    assert sorted(back, key=lambda r: (r.experiment, r.n)) == sorted(recs, key=lambda r: (r.experiment, r.n))
    bad = tmp_path / "bad.csv"
    bad.write_text("nope\n")
    with pytest.raises(ValueError):
        bc.load_records(str(bad))


def test_exit_code_2_without_backend(capsys, monkeypatch):
    monkeypatch.setattr(bc, "native_unavailable_reason", lambda: "no CUDA device visible")
    assert bc.main(["--experiment", "fullsort", "--type", "i32", "--max-exp", "3", "--reps", "1"]) == 2
    assert "unavailable" in capsys.readouterr().err


def test_gate_raises_on_mismatch():
    with pytest.raises(bc.GateError):
        bc._gate("x", "00", "11")
    assert bc._gate("x", "11", "11") == "11"


@pytest.mark.gpu
def test_benchcli_gpu_matches_reference_checksums(tmp_path):
    out = tmp_path / "b200.csv"
    rc = bc.main(["--max-exp", "14", "--reps", "1", "--out", str(out)])
    assert rc == 0
    got = bc.load_records(str(out))
    gold = _golden()
    assert {(r.experiment, r.elem_type, r.n, r.algorithm) for r in got} == set(gold)
    for r in got:
        assert r.checksum == gold[(r.experiment, r.elem_type, r.n, r.algorithm)], r
        assert r.mean_seconds > 0


@pytest.mark.gpu
def test_benchcli_gate_catches_wrong_output(monkeypatch, capsys):
    import paper_1704_08579_b200.benchcli as mod

    def broken(region, config):
        region.zero_()

    monkeypatch.setattr(mod, "sort_with_config", broken)
    assert mod.main(["--experiment", "fullsort", "--type", "i32", "--max-exp", "4", "--reps", "1"]) == 1
    assert "correctness gate failed" in capsys.readouterr().err
