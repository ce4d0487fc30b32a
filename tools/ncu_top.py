"""Per-source-line instruction / stall shares of one kernel in an ncu report.

    python tools/ncu_top.py REPORT.ncu-rep KERNEL_REGEX [top] [launch_skip]
"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
skip = sys.argv[4] if len(sys.argv) > 4 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}", "--launch-skip", skip,
                      "--launch-count", "1", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows, hdr, f = [], None, None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "Function Name":
        continue
    d = dict(zip(hdr, r))
    try:
        ie = int(d.get("Instructions Executed") or 0)
        ws = int(d.get("Warp Stall Sampling (All Samples)") or 0)
    except ValueError:
        continue
    if r[0] and r[0] != "-" and r[1]:
        rows.append((ie, ws, f, r[0], r[1][:85]))
ti = sum(x[0] for x in rows) or 1
tw = sum(x[1] for x in rows) or 1
print(f"{kre}: {ti:,} warp-inst, {tw:,} stall samples")
for x in sorted(rows, key=lambda x: -x[0])[:top]:
    print(f"  {100*x[0]/ti:5.1f}%i {100*x[1]/tw:5.1f}%s {x[2]}:{x[3]} {x[4]}")
