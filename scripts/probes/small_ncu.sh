#!/bin/bash
for s in 256,256,2,50%,32,14,14 1024,1024,8,50%,32,14,14; do
  echo "== $s"
  SCC_SHAPE=$s timeout 60 python scripts/probes/small_ops.py
  SCC_SHAPE=$s EAGER=1 timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/probes/small_ops.py 2>/dev/null | grep -v "^==" | python -c "
import sys, csv, collections
rows = list(csv.reader(sys.stdin))
hdr = rows[0]; ki = hdr.index('Kernel Name'); vi = hdr.index('Metric Value')
seq = [(r[ki][:60], float(r[vi])) for r in rows[1:] if len(r) > vi]
for k, v in seq[-24:]: print(f'  {v/1e3:8.2f} us  {k}')
"
done
