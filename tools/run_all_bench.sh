#!/bin/bash
# Runs every bench workload on one GPU (plus the reference arm of the
# default) and writes JSON lines to gpurun_out/all/.  Usage (on the box):
#   bash tools/run_all_bench.sh [steps] [warmup]
S=${1:-5}; W=${2:-3}
mkdir -p gpurun_out/all
timeout 900 python bench.py --steps $S --warmup $W > gpurun_out/all/default.json 2> gpurun_out/all/default.err
echo "default rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/all/reference.json 2> gpurun_out/all/reference.err
echo "reference rc=$?"
for w in sort_i32 sort_f64 c1 c2_i32 c2_f64 c3 c4 c5_f64_uniform; do
  timeout 600 python bench.py --workload $w --steps $S --warmup $W > gpurun_out/all/$w.json 2> gpurun_out/all/$w.err
  echo "$w rc=$?"
done
for t in i32 f64; do for d in sorted reverse few; do
  timeout 600 python bench.py --workload c5_${t}_$d --steps $S --warmup $W --no-e2e > gpurun_out/all/c5_${t}_$d.json 2> gpurun_out/all/c5_${t}_$d.err
  echo "c5_${t}_$d rc=$?"
done; done
python - <<'PY'
import glob, json, os
for f in sorted(glob.glob("gpurun_out/all/*.json")):
    try:
        d = json.load(open(f))
    except Exception as e:
        print(os.path.basename(f), "FAILED", e); continue
    r = d.get("roofline", {})
    print(f"{os.path.basename(f):24s} value={d.get('value',0):9.3f} ms={d.get('ms_per_step',0):9.3f} "
          f"frac={r.get('frac')} kern={r.get('kernel')} e2e={d.get('e2e',{}).get('value')} "
          f"cpu={d.get('cpu_baseline',{}).get('value')} clocks={d.get('clocks',{}).get('sm_mhz')}")
PY
