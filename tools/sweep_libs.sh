# A/B timing of alternative builds of the library (VEXSORT_B200_LIB override).
#   bash tools/sweep_libs.sh LIB.so [LIB.so ...]   (WORKLOADS env: default "sort_i32 sort_f64")
for L in "$@"; do for w in ${WORKLOADS:-sort_i32 sort_f64}; do VEXSORT_B200_LIB=$L timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(\"$L\", \"$w\", round(d[\"ms_per_step\"],3), {k:round(v[\"ms\"]/d[\"steps\"],3) for k,v in d[\"kernels\"].items()})"; done; done
