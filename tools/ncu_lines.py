"""Top source lines of one kernel in an ncu report (instructions executed and
warp-stall samples), from `ncu --page source --print-source cuda,sass`.

    python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [launch_skip] [top]
"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}", "--launch-skip", skip,
                      "--launch-count", "1", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows, cur_file, hdr = [], None, None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] in ("Function Name",):
        continue
    d = dict(zip(hdr, r))
    try:
        ie = int(d.get("Instructions Executed") or 0)
        ws = int(d.get("Warp Stall Sampling (All Samples)") or 0)
    except ValueError:
        continue
    rows.append((ie, ws, f"{cur_file}:{r[0]}", r[1][:80]))
ti = sum(x[0] for x in rows) or 1
tw = sum(x[1] for x in rows) or 1
print(f"total warp-instructions {ti:,}  stall samples {tw:,}")
print("-- by stall samples")
for ie, ws, loc, src in sorted(rows, key=lambda x: -x[1])[:top]:
    print(f"{100*ws/tw:5.1f}% stall {100*ie/ti:5.1f}% inst  {loc:22s} {src}")
