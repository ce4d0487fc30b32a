#!/bin/bash
# Memory-safety evidence without compute-sanitizer (closed on this pool): the
# GPU parity + canary tests against a -DVX_CHECK build, whose kernels assert
# every bucket index, staging slot and destination index on the device (a
# failed assertion traps and fails the launch).  Build build/check.so first:
#   bash tools/build_variant.sh check -DVX_CHECK
# Output: gpurun_out/check/ (copy to profiles/sanitizer_rNN/).
mkdir -p gpurun_out/check
export VEXSORT_B200_LIB=$PWD/build/check.so
python - <<'PY' > gpurun_out/check/lib.txt 2>&1
import paper_1704_08579_b200 as vx
print("library under test:", vx._lib.lib_path())
PY
timeout ${CHECK_TIMEOUT:-1500} python -m pytest tests -m gpu -q --timeout 900 \
  -k "${TESTK:-not sharded and not integration}" > gpurun_out/check/pytest_vx_check.log 2>&1
echo "VX_CHECK build: pytest rc=$? $(tail -1 gpurun_out/check/pytest_vx_check.log)"
for w in sort_i32 sort_f64 c4 c2_i32 c3 c5_i32_sorted c5_f64_few; do
  timeout 600 python bench.py --workload $w --steps 1 --warmup 1 --no-cpu --no-e2e 2>&1 | \
    python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$w', 'verified', d.get('verified'), d['ms_per_step'], 'ms')" \
    >> gpurun_out/check/bench_vx_check.log 2>&1
done
cat gpurun_out/check/bench_vx_check.log
