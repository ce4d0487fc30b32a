#!/bin/bash
# compute-sanitizer over tools/sanitize_cases.py on the GPU box; logs land in
# gpurun_out/sanitizer/ (copy them to profiles/sanitizer_rNN/).
#   bash tools/sanitize.sh [tools...]   (default: memcheck racecheck synccheck initcheck)
OUT=gpurun_out/sanitizer
mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in ${@:-memcheck racecheck synccheck initcheck}; do
  extra=""
  mode=full
  case $tool in
    racecheck) extra="--racecheck-report all" ;;
    initcheck) extra="--track-unused-memory no"; mode=quick ;;
  esac
  timeout ${SAN_TIMEOUT:-1500} $CS --tool $tool $extra --print-limit 50 --error-exitcode 9 \
    --kernel-name regex:"(qs_|partition2|segsort|bp_|select_splitters)" \
    python tools/sanitize_cases.py $mode > $OUT/$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $OUT/$tool.log | tail -1)"
done
