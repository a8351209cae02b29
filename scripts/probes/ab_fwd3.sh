#!/bin/bash
# c1 forward and step, alternating on one box: in-tree vs build/pre_dsc
for i in 1 2 3; do
  for lib in "" build/pre_dsc; do
    if [ -n "$lib" ]; then export SCC_LIB_PATH=$lib/libscc_b200.so; else unset SCC_LIB_PATH; fi
    b=$(timeout 300 python bench.py --steps 200 --warmup 10 --no-e2e --no-cpu-baseline --no-models --no-compositions --no-c5 --no-traffic 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['kernel_ms'])")
    echo "${lib:-intree}: $(timeout 120 python scripts/band_timing.py 32 64 128 32 32 2 x 2>&1 | head -2 | tr '\n' ' ') | bench $b"
  done
done
