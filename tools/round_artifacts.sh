#!/bin/bash
# Round-end evidence on the GPU box, sized to come back through gpurun
# (< 64 MiB): GPU tests + smoke, every bench line, the launch list of the
# default bench, full ncu captures summarised ON THE BOX (only the sort_i32
# report is kept).  Outputs land in gpurun_out/art/.
#   bash tools/round_artifacts.sh TAG
TAG=${1:-r1}
mkdir -p gpurun_out/art
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/art/pytest_gpu.log 2>&1
echo "pytest rc=$? $(tail -1 gpurun_out/art/pytest_gpu.log)"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/art/smoke.log 2>&1
echo "smoke rc=$?"
bash tools/run_all_bench.sh 5 3
cp gpurun_out/all/*.json gpurun_out/art/ 2>/dev/null
FULL_TIMEOUT=500 bash tools/profile_round.sh sort_i32 sort_f64 c4 c3 c2_i32
bash tools/headline_traffic.sh c5_i32_uniform c5_f64_uniform
python tools/summarize_ncu.py --full gpurun_out/prof/full_sort_i32.ncu-rep:sort_i32 \
  gpurun_out/prof/full_sort_f64.ncu-rep:sort_f64 gpurun_out/prof/full_c4.ncu-rep:c4 \
  gpurun_out/prof/full_c3.ncu-rep:c3 gpurun_out/prof/full_c2_i32.ncu-rep:c2_i32 \
  --traffic gpurun_out/traffic/c5_i32_uniform.ncu-rep:c5_i32_uniform gpurun_out/traffic/c5_f64_uniform.ncu-rep:c5_f64_uniform \
  --launches gpurun_out/prof/launches_default.csv --tag $TAG > gpurun_out/art/summarize.log 2>&1
echo "summarize rc=$?"
cp profiles/ncu_summary_$TAG.md profiles/ncu_traffic.json gpurun_out/art/ 2>/dev/null
cp gpurun_out/prof/launches_default.csv gpurun_out/art/launches_default_$TAG.csv
for w in sort_i32 sort_f64 c4 c3 c2_i32; do python tools/ncu_stalls.py gpurun_out/prof/full_$w.ncu-rep > gpurun_out/art/stalls_$w.txt 2>&1; done
# (the .ncu-rep files stay on the box: gpurun brings back at most 64 MiB)
rm -rf gpurun_out/prof gpurun_out/all gpurun_out/quick gpurun_out/traffic
