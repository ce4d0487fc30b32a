#!/bin/bash
# sort time vs n for tuning the small-size path:  ENVV="A=1 B=2" bash tools/small_sweep.sh "20 21 22 23 24"
for e in ${1:-20 21 22 23 24}; do
  env $ENVV timeout 300 python bench.py --workload sort_i32 --n "2**$e" --steps 20 --warmup 5 --no-e2e --no-cpu 2>/dev/null | \
    python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$ENVV', 'n=2^$e', round(d['ms_per_step'],4), 'ms', {k:v['ms_per_step'] for k,v in d['kernels'].items()}, d.get('verified'))"
done
