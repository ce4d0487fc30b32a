"""Copy a round's artifacts from gpurun_out/art into profiles/, look the
dominant kernels' DRAM traffic up in the same run's ncu capture, and replace
the status table of DESIGN.md.   python tools/refresh_profiles.py r2"""
import glob
import json
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
tag = sys.argv[1] if len(sys.argv) > 1 else "r2"
A = os.path.join(ROOT, "gpurun_out", "art")
B = os.path.join(ROOT, "profiles", f"bench_{tag}")
os.makedirs(B, exist_ok=True)
for f in glob.glob(os.path.join(A, "*.json")):
    if os.path.basename(f) != "ncu_traffic.json":
        shutil.copy(f, B)
shutil.copy(os.path.join(A, "pytest_gpu.log"), B)
for f in (f"ncu_summary_{tag}.md", "ncu_traffic.json", f"launches_default_{tag}.csv"):
    shutil.copy(os.path.join(A, f), os.path.join(ROOT, "profiles"))
os.makedirs(os.path.join(ROOT, "profiles", f"stalls_{tag}"), exist_ok=True)
for f in glob.glob(os.path.join(A, "stalls_*.txt")):
    shutil.copy(f, os.path.join(ROOT, "profiles", f"stalls_{tag}"))
import bench  # noqa: E402

for f in sorted(glob.glob(os.path.join(B, "*.json"))):
    d = json.load(open(f))
    r = d.get("roofline")
    if not r or "kernels" not in d:
        continue
    k = r["kernel"].split(" ")[0]
    if k not in bench.CLASSES:
        continue
    t = bench.ncu_traffic(d["config"]["workload"], k)
    if t and r.get("alg_bytes_per_launch"):
        r["traffic"] = t
        r["traffic_over_alg"] = round(t / r["alg_bytes_per_launch"], 3)
        r["traffic_note"] = ("looked up in profiles/ncu_traffic.json of the same artifact run (the capture follows "
                             "the bench lines in tools/round_artifacts.sh)")
        json.dump(d, open(f, "w"))
table = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "design_table.py"), B], capture_output=True,
                       text=True).stdout
p = os.path.join(ROOT, "DESIGN.md")
s = open(p).read()
i = s.index("| config | workload | ms / step | Gelem/s | passes-equiv.")
j = s.index("Round-2 progression of the default line")
open(p, "w").write(s[:i] + table + "\n" + s[j:])
print(table)
print(open(os.path.join(B, "pytest_gpu.log")).read().strip().splitlines()[-1])
print(open(os.path.join(A, "smoke.log")).read().strip().splitlines()[-1])
