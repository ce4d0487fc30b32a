"""Warp-stall breakdown (PC sampling) per kernel of an ncu report.

    python tools/ncu_stalls.py REPORT.ncu-rep
"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    items = []
    for k, v in d.items():
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
            try:
                items.append((k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v)))
            except ValueError:
                pass
    tot = sum(v for _, v in items) or 1
    items.sort(key=lambda x: -x[1])
    print(d["Kernel Name"][:60], d.get("gpu__time_duration.sum"))
    print("   " + ", ".join(f"{k} {100*v/tot:.0f}%" for k, v in items[:9]))
