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
# The partition's build option VX_PART_LOOKBACK (tile-ordered, run-to-run
# identical layout by decoupled look-back): the partition tests against that
# build, plus a determinism check of the layout.
#   bash tools/build_variant.sh lookback -DVX_PART_LOOKBACK
if [ -f build/lookback.so ]; then
  export VEXSORT_B200_LIB=$PWD/build/lookback.so
  timeout 900 python -m pytest tests -m gpu -q --timeout 600 -k "partition or c3" > gpurun_out/check/pytest_lookback.log 2>&1
  echo "VX_PART_LOOKBACK build: pytest rc=$? $(tail -1 gpurun_out/check/pytest_lookback.log)"
  python - <<'PY' >> gpurun_out/check/pytest_lookback.log 2>&1
import numpy as np, torch
import paper_1704_08579_b200 as vx
x = torch.from_numpy(np.random.default_rng(3).standard_normal((1 << 24) + 77)).cuda()
outs = []
for _ in range(3):
    t = x.clone()
    b = vx.partition_region(t, 0.1)
    outs.append(t)
assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2]), "look-back layout differs between runs"
print("look-back layout identical over 3 runs, split", b)
PY
  tail -1 gpurun_out/check/pytest_lookback.log
fi
