#!/bin/bash
# Regenerates tests/golden/benchcli_ref_checksums.csv from the REFERENCE's
# own bench CLI (vexsort/benchcli.py, native backend) -- run in the build
# container only (needs /root/reference; copied to /tmp because the tree is
# read-only).  Timings are dropped: only the deterministic columns are kept.
set -e
rm -rf /tmp/vexref && cp -r /root/reference/pkg /tmp/vexref
(cd /tmp && PYTHONPATH=/tmp/vexref/src python -m vexsort.benchcli --max-exp 14 --reps 1 --backend native \
  --out /tmp/benchcli_ref.csv)
python - <<'PY'
import csv, os
here = os.path.dirname(os.path.abspath("tests/golden/x"))
rows = list(csv.DictReader(open("/tmp/benchcli_ref.csv")))
with open(os.path.join(here, "benchcli_ref_checksums.csv"), "w") as f:
    f.write("experiment,elem_type,n,algorithm,checksum\n")
    for r in rows:
        f.write(f"{r['experiment']},{r['elem_type']},{r['n']},{r['algorithm']},{r['checksum']}\n")
PY
