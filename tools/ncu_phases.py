"""Instruction / stall share per source file and per line range of one kernel.

    python tools/ncu_phases.py REPORT.ncu-rep KERNEL_REGEX SKIP file:lo-hi=name ...
"""
import csv
import io
import subprocess
import sys

rep, kre, skip = sys.argv[1], sys.argv[2], sys.argv[3]
ranges = []
for a in sys.argv[4:]:
    loc, name = a.split("=")
    f, lh = loc.split(":")
    lo, hi = lh.split("-")
    ranges.append((f, int(lo), int(hi), name))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}", "--launch-skip", skip,
                      "--launch-count", "1", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
hdr, f = None, None
agg, byfile, tot = {}, {}, [0, 0]
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "Function Name" or not r[0] or r[0] == "-" or not r[1]:
        continue
    d = dict(zip(hdr, r))
    try:
        ln = int(r[0])
        ie = int(d.get("Instructions Executed") or 0)
        ws = int(d.get("Warp Stall Sampling (All Samples)") or 0)
    except ValueError:
        continue
    tot[0] += ie
    tot[1] += ws
    bf = byfile.setdefault(f, [0, 0])
    bf[0] += ie
    bf[1] += ws
    for (rf, lo, hi, name) in ranges:
        if rf == f and lo <= ln <= hi:
            a = agg.setdefault(name, [0, 0])
            a[0] += ie
            a[1] += ws
print(f"total {tot[0]:,} warp-inst, {tot[1]:,} samples")
for k, (i, w) in sorted(byfile.items(), key=lambda x: -x[1][0]):
    print(f"  file {k:32s} {100*i/tot[0]:5.1f}%i {100*w/max(tot[1],1):5.1f}%s")
for k, (i, w) in agg.items():
    print(f"  {k:24s} {100*i/tot[0]:5.1f}%i {100*w/max(tot[1],1):5.1f}%s")
