#!/bin/bash
# DRAM bytes + duration per launch of ONE step of the headline workloads
# (2^32 int32 / 2^31 float64): three metrics only -- a --set full capture
# would replay every 16 GiB launch ~40 times.  Each capture runs only after
# the same bench command exited 0 without ncu.
#   bash tools/headline_traffic.sh [workloads...]   -> gpurun_out/traffic/
mkdir -p gpurun_out/traffic
for w in ${@:-c5_i32_uniform c5_f64_uniform}; do
  timeout 600 python bench.py --workload $w --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/traffic/$w.plain.json 2> gpurun_out/traffic/$w.plain.err \
    || { echo "$w: plain run failed"; continue; }
  timeout ${NCU_TIMEOUT:-1500} ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k 'regex:(qs_|partition2|segsort|bp_)' -o gpurun_out/traffic/$w -f \
    python bench.py --workload $w --steps 1 --warmup 0 --prof-steps 1 --no-e2e --no-cpu > gpurun_out/traffic/$w.log 2>&1
  echo "traffic $w rc=$? $(ls -la gpurun_out/traffic/$w.ncu-rep 2>/dev/null | awk '{print $5}') bytes"
done
