#!/bin/bash
# A/B of environment knobs on bench workloads (output: knobs workload ms kernels)
#   W="sort_i32 c5_i32_uniform" bash tools/env_ab.sh "" "VX_HIST_WAVES=2" "VX_HIST_WAVES=4 VX_SCAT_WAVES=2"
mkdir -p gpurun_out/eab
for r in $(seq ${R:-1}); do for E in "$@"; do for w in ${W:-sort_i32}; do
  f=gpurun_out/eab/out.json
  env $E timeout 300 python bench.py --workload $w --steps ${S:-5} --warmup 3 --no-e2e --no-cpu > $f 2> gpurun_out/eab/out.err
  python -c "import json,sys; d=json.load(open('$f')); print('[$E]', '$w', round(d['ms_per_step'],3), d['verified'], {k:round(v['ms_per_step'],3) for k,v in d.get('kernels',{}).items() if v['ms_per_step']>0.05})" 2>&1 | tail -1
done; done; done
