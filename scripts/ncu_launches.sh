#!/bin/bash
# Launch list (per-kernel device time + DRAM bytes) of our kernels in one
# short bench run.  Usage: scripts/ncu_launches.sh OUT.csv [bench args...]
out=$1; shift
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:'scc|band|weight|tc_' -c 40 --csv --log-file "$out" \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-models --no-c5 "$@" > /dev/null 2>&1
python - "$out" <<'PY'
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[0].isdigit()]
agg = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows:
    name = r[4].split("(")[0][-60:]
    agg[name][r[-3]].append(float(r[-1].replace(",", "")))
for k, m in agg.items():
    t = m.get("gpu__time_duration.sum", [0]); rd = m.get("dram__bytes_read.sum", [0]); wr = m.get("dram__bytes_write.sum", [0])
    print(f"{k:60s} n={len(t):3d} avg_us={sum(t)/len(t)/1e3:8.2f} rdMB={sum(rd)/len(rd)/1e6:7.2f} wrMB={sum(wr)/len(wr)/1e6:7.2f}")
PY
