#!/bin/bash
# A/B (alternating, one box): in-tree library vs $1: c1 forward, the 64->64
# N=128 32x32 forward, and the c1 bench step
for i in 1 2 3; do
  for lib in "" $1; do
    if [ -n "$lib" ]; then export SCC_LIB_PATH=$lib/libscc_b200.so; else unset SCC_LIB_PATH; fi
    b=$(timeout 300 python bench.py --steps 200 --warmup 10 --no-e2e --no-cpu-baseline --no-models --no-compositions --no-c5 --no-traffic 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['kernel_ms']['forward'])")
    f1=$(timeout 120 python scripts/band_timing.py 32 64 128 32 32 2 x 2>&1 | head -1)
    f2=$(timeout 120 python scripts/band_timing.py 128 64 64 32 32 2 x 2>&1 | head -1)
    echo "${lib:-intree}: c1 $f1 | 64->64 N128 $f2 | bench $b"
  done
done
