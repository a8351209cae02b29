#!/bin/bash
# depthwise kernels: in-tree vs $1 (scripts/dsc_timing.py columns of our kernels)
for i in 1 2; do for lib in "" $1; do
  if [ -n "$lib" ]; then export SCC_LIB_PATH=$lib/libscc_b200.so; else unset SCC_LIB_PATH; fi
  echo "${lib:-intree}"
  python scripts/dsc_timing.py 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print(' ', d['c_in'], d['hw'], d['stride'], 'fwd', d['dw_ours_us'], 'bdata', d['dw_bwd_data_ours_us'], 'one', d['dw_bwd_ours_us'], 'pair', d['pair_ours_us'])
"
done; done
