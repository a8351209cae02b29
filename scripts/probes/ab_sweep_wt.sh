#!/bin/bash
# C5 co=50% rows: this tree vs the worktree at build/wt_r02c (alternating, one box)
mkdir -p gpurun_out
for i in 1 2; do
  for d in . build/wt_r02c; do
    (cd $d && timeout 600 python scripts/sweep.py --co 50 --out /tmp/sw.json > /dev/null 2>&1)
    python - "$d" <<'PY'
import json, sys
r = json.load(open("/tmp/sw.json"))["rows"]
print(sys.argv[1].ljust(14), " ".join(f"{x['C']}/{x['hw']}/{x['cg']}:{x['us']['step']:.1f}" for x in r))
PY
  done
done
