#!/bin/bash
# A/B: current library vs scripts/probes/_ab (an older build) on sweep subsets, interleaved
for rep in 1 2; do
  for lib in new old; do
    if [ $lib = old ]; then export SCC_LIB_PATH=$PWD/scripts/probes/_ab/libscc_b200.so; else unset SCC_LIB_PATH; fi
    echo "== $lib rep $rep"
    timeout 300 python scripts/sweep.py --C 256 512 --cg 2 8 --co 50 --hw 14 --parts 2>&1 | grep '"C"' | python -c "
import sys, json
for l in sys.stdin:
    r = json.loads(l); print(r['C'], r['cg'], r['co'], r['hw'], r['us'])"
  done
done
