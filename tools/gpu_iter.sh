# iteration loop on the GPU box: GPU tests (filter in $TESTK), then bench lines
#   TESTK="expr" WL="w1 w2" AB=1 bash tools/gpu_iter.sh
mkdir -p gpurun_out/it
timeout ${PYT_TIMEOUT:-1200} python -m pytest tests -m gpu -x -q --timeout ${TEST_TIMEOUT:-600} -k "${TESTK:-not c5_full_size}" > gpurun_out/it/pytest.log 2>&1
echo "pytest rc=$? $(tail -1 gpurun_out/it/pytest.log)"
grep -E "^E |FAILED|Error" gpurun_out/it/pytest.log | head -20
for w in ${WL-c5_i32_uniform sort_i32}; do
  for v in ${VARIANTS:-default}; do
    env=""; [ "$v" != default ] && env="$v=1"
    env $env timeout 600 python bench.py --workload $w --steps ${STEPS:-5} --warmup 3 --no-cpu --no-e2e > gpurun_out/it/$w.$v.json 2> gpurun_out/it/$w.$v.err
    rc=$?
    python - "$w" "$v" "$rc" <<'PY'
import json, sys
w, v, rc = sys.argv[1:]
try:
    d = json.load(open(f"gpurun_out/it/{w}.{v}.json"))
except Exception as e:
    print(w, v, "FAILED rc", rc, open(f"gpurun_out/it/{w}.{v}.err").read()[-800:]); sys.exit()
ks = {k: v2["ms_per_step"] for k, v2 in d["kernels"].items()}
print(f"{w:16s} {v:14s} {d['value']:8.2f} Gelem/s {d['ms_per_step']:8.3f} ms ver={d['verified']} {ks} {d.get('sort_stats',{}).get('scatter_levels_per_key')}")
PY
  done
done
