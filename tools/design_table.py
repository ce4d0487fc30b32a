"""Markdown status table for DESIGN.md from the bench lines of a round:
    python tools/design_table.py profiles/bench_r2"""
import json
import os
import sys

d = sys.argv[1] if len(sys.argv) > 1 else "profiles/bench_r2"
rows = [("default", "C5 (default)", "int32 2^32 uniform, 1 GPU"), ("c5_i32_sorted", "C5", "int32 2^32 sorted"),
        ("c5_i32_reverse", "C5", "int32 2^32 reverse"), ("c5_i32_few", "C5", "int32 2^32 few-unique"),
        ("c5_f64_uniform", "C5", "float64 2^31 uniform"), ("c5_f64_sorted", "C5", "float64 2^31 sorted"),
        ("c5_f64_reverse", "C5", "float64 2^31 reverse"), ("c5_f64_few", "C5", "float64 2^31 few-unique"),
        ("sort_i32", "north-star", "int32 2^28 sort"), ("sort_f64", "—", "float64 2^28 sort"),
        ("c1", "C1", "int32 2^20 sort"), ("c2_i32", "C2", "2^20 segments, int32"),
        ("c2_f64", "C2", "2^20 segments, float64"), ("c3", "C3", "float64 2^28 partition"), ("c4", "C4", "kv 2^28")]
print("| config | workload | ms / step | Gelem/s | passes-equiv. | dominant kernel (frac of HBM peak; DRAM traffic / alg.) | "
      "e2e Gelem/s (pipelined / single call) | CPU port Gelem/s (cores) / 1 core / numba reference 1 core |")
print("|---|---|---|---|---|---|---|---|")
for f, cfg, wl in rows:
    p = os.path.join(d, f + ".json")
    if not os.path.exists(p):
        continue
    j = json.load(open(p))
    r = j["roofline"]
    k = r["kernel"].split(" ")[0] if not r["kernel"].startswith("whole") else "whole sort (latency-bound)"
    tr = r.get("traffic_over_alg")
    e = j.get("e2e") or {}
    sc = e.get("single_call") or {}
    e2e = "—" if not e else (f"{e['value']:.2f} / {sc['value']:.2f}" if sc else f"{e['value']:.2f}")
    cb = j.get("cpu_baseline") or {}
    s1 = (cb.get("single_core") or {}).get("value")
    nb = (cb.get("reference_numba") or {}).get("value")
    cpu = f"{cb.get('value', 0):.4f} ({cb.get('cores')})" + (f" / {s1:.4f}" if s1 else " / —") + (f" / {nb:.4f}" if nb else " / —")
    print(f"| {cfg} | {wl} | {j['ms_per_step']:.3f} | {j['value']:.1f} | {j['step_roofline']['passes_equiv']} | "
          f"{k} ({r['frac']:.2f}{'; ' + str(tr) + 'x' if tr else ''}) | {e2e} | {cpu} |")
