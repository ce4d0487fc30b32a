#!/bin/bash
# ncu evidence for profiles/ (run on the GPU box, one GPU; each capture only
# after the same command exited 0 without ncu -- run_all_bench.sh first).
#   bash tools/profile_round.sh [workloads...]
# 1. launch list of the default bench command (gpu__time_duration, serialised)
#    -- skipped when NO_LAUNCHES=1
# 2. per workload: --set full of every launch of ONE step (steps 1, warmup 0).
#    Keep to the 2^28 workloads: a full capture replays every kernel ~40x and
#    saves/restores the buffers it writes, which at 2^32 (16 GiB) takes hours.
mkdir -p gpurun_out/prof
WL=${@:-sort_i32 sort_f64 c3 c2_i32 c4}
if [ "${NO_LAUNCHES:-0}" != 1 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/prof/launches_default.csv python bench.py --steps 2 --warmup 3 --no-cpu \
    > gpurun_out/prof/launches_default.log 2>&1
  echo "launch list rc=$?"
fi
for w in $WL; do
  timeout ${FULL_TIMEOUT:-600} ncu --set full --import-source on --clock-control none -k 'regex:(qs_|partition2|segsort|bp_)' \
    -o gpurun_out/prof/full_$w -f python bench.py --workload $w --steps 1 --warmup 0 --no-e2e --no-cpu \
    > gpurun_out/prof/full_$w.log 2>&1
  echo "full $w rc=$?"
done
