#!/bin/bash
# A/B (alternating, same box) of the gen-1 launch chaining variants on the
# 14x14 C5 rows + two 56x56 rows: in-tree library vs build/ab_{trig,pdl,both}
mkdir -p gpurun_out
run() {  # $1 label, $2 lib dir or ""
  if [ -n "$2" ]; then export SCC_LIB_PATH=$2/libscc_b200.so; else unset SCC_LIB_PATH; fi
  timeout 300 python scripts/sweep.py --co 50 --C 256 1024 --hw 14 --out gpurun_out/ab_$1.json > /dev/null 2>&1
  timeout 300 python scripts/sweep.py --co 50 --C 512 --cg 4 --hw 56 --out gpurun_out/ab56_$1.json > /dev/null 2>&1
  python - "$1" <<'PY'
import json, sys
l = sys.argv[1]
r = json.load(open(f"gpurun_out/ab_{l}.json"))["rows"] + json.load(open(f"gpurun_out/ab56_{l}.json"))["rows"]
print(l.ljust(6), " ".join(f"{x['C']}/{x['hw']}/{x['cg']}: {x['us']['fwd']:.1f} {x['us']['bwd']:.1f} {x['us']['step']:.1f}" for x in r))
PY
}
for i in 1 2; do
  run cur ""
  run trig build/ab_trig
  run pdl build/ab_pdl
  run both build/ab_both
done
