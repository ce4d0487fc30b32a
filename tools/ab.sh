#!/bin/bash
# A/B of library builds on one workload, R rounds (output: lib workload ms kernels)
#   W=c3 R=2 bash tools/ab.sh build/a.so build/b.so ...
mkdir -p gpurun_out/ab
for r in $(seq ${R:-2}); do for L in "$@"; do for w in ${W:-c3}; do
  f=gpurun_out/ab/$(basename $L .so)_$w.json
  VEXSORT_B200_LIB=$L timeout 300 python bench.py --workload $w --steps ${S:-5} --warmup 3 --no-e2e --no-cpu > $f 2> ${f%.json}.err
  python -c "import json,sys; d=json.load(open('$f')); print('$L', '$w', round(d['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in d.get('kernels',{}).items()})" 2>&1 | tail -1
done; done; done
