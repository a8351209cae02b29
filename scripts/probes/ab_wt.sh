#!/bin/bash
# c1 forward / step: this tree vs the worktree at build/wt_r02c (alternating, one box)
for i in 1 2 3; do
  for d in . build/wt_r02c; do
    b=$(cd $d && timeout 300 python bench.py --steps 200 --warmup 10 --no-e2e --no-cpu-baseline --no-models --no-compositions --no-c5 --no-traffic 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['kernel_ms'])")
    echo "$d: $(cd $d && timeout 120 python scripts/band_timing.py 32 64 128 32 32 2 x 2>&1 | head -1) | bench $b"
  done
done
