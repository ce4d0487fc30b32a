"""Executed instructions and stall samples per SASS opcode of one kernel.

    python tools/ncu_sass_ops.py REPORT.ncu-rep KERNEL_REGEX [launch_skip] [top]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep, kre = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}", "--launch-skip", skip,
                      "--launch-count", "1", "--print-source", "sass"], capture_output=True, text=True).stdout
hdr = None
ops = defaultdict(lambda: [0, 0])
tot = [0, 0]
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "Address":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) - 2 or not r[0].startswith("0x"):
        continue
    d = dict(zip(hdr, r))
    src = d["Source"].strip()
    if src.startswith("@"):
        src = src.split(None, 1)[1]
    op = src.split()[0]
    base = ".".join(op.split(".")[:2]) if op.split(".")[0] in ("IMAD", "LDS", "STS", "LDG", "STG", "SHFL", "ATOMS") else op.split(".")[0]
    try:
        ie = int(d["Instructions Executed"])
        ws = int(d["Warp Stall Sampling (All Samples)"])
    except ValueError:
        continue
    ops[base][0] += ie
    ops[base][1] += ws
    tot[0] += ie
    tot[1] += ws
print(f"total warp-instructions {tot[0]:,}  stall samples {tot[1]:,}")
for k, (ie, ws) in sorted(ops.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{k:18s} inst {100 * ie / max(tot[0], 1):5.1f}%  stall {100 * ws / max(tot[1], 1):5.1f}%  ({ie:,})")
