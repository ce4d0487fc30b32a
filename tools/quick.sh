#!/bin/bash
# Iteration loop on the GPU box: parity tests, then a few bench workloads.
#   bash tools/quick.sh [workloads...]   (default: sort_i32 sort_f64 c4)
mkdir -p gpurun_out/quick
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/quick/pytest.log 2>&1
echo "pytest rc=$? $(tail -1 gpurun_out/quick/pytest.log)"
for w in ${@:-sort_i32 sort_f64 c4}; do
  timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/quick/$w.json 2> gpurun_out/quick/$w.err
  python - "$w" <<'PY'
import json, sys
w = sys.argv[1]
try:
    d = json.load(open(f"gpurun_out/quick/{w}.json"))
except Exception as e:
    print(w, "FAILED", e); sys.exit()
ks = {k: round(v["ms"] / d["steps"], 3) for k, v in d["kernels"].items()}
print(f"{w:16s} {d['value']:8.2f} Gelem/s {d['ms_per_step']:8.3f} ms  {ks}")
PY
done
