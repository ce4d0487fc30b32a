mkdir -p gpurun_out/r2a
timeout 900 python -m pytest tests -m gpu -x -q -k "not c5_full_size" > gpurun_out/r2a/pytest.log 2>&1
echo "pytest rc=$? $(tail -1 gpurun_out/r2a/pytest.log)"
for w in c5_i32_uniform c1 sort_i32 c4; do
  timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu $( [ $w != c5_i32_uniform ] && echo --no-e2e ) > gpurun_out/r2a/$w.json 2> gpurun_out/r2a/$w.err
  echo "$w rc=$? $(head -c 600 gpurun_out/r2a/$w.json)"
done
