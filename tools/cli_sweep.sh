#!/bin/bash
# vexsort vs torch.sort through the bench CLI (fresh buffers every repetition, host time included)
#   bash tools/cli_sweep.sh [type] [max_exp]
python -m paper_1704_08579_b200.benchcli --experiment fullsort --type ${1:-i32} --max-exp ${2:-26} --reps 7 2>/dev/null | \
  python -c "
import sys
rows={}
for l in sys.stdin:
    if not l.startswith('fullsort'): continue
    f=l.strip().split(',')
    rows.setdefault(int(f[2]),{})[f[3]]=float(f[5])*1e3
for n in sorted(rows):
    r=rows[n]; print(f'n={n:>10d}  vexsort {r.get(\"vexsort\",0):.4f} ms  torch.sort {r.get(\"baseline_sort\",0):.4f} ms  ratio {r.get(\"baseline_sort\",0)/max(r.get(\"vexsort\",1e-9),1e-9):.2f}')
"
