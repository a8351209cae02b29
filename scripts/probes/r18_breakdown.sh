#!/bin/bash
# SCC-ResNet-18 (batch 128) kernel-time breakdown from an ncu launch list (cold, serialised)
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof_r18.csv python scripts/model_profile.py resnet18 > /dev/null 2>&1
python - gpurun_out/prof_r18.csv <<'PY'
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[0].isdigit()]
agg = collections.Counter(); cnt = collections.Counter(); tot = 0
for r in rows:
    v = float(r[-1].replace(",", "")); tot += v
    n = r[4]
    k = ("scc:" + n.split("(")[0].replace("void ", "")[-60:]) if "scc::" in n else ("torch:" + n.split("(")[0][-50:])
    agg[k] += v; cnt[k] += 1
print(f"total {tot/1e3:.1f} us over {len(rows)} kernels")
for k, v in agg.most_common(22): print(f"{v/1e3:9.1f} us {100*v/tot:5.1f}% n={cnt[k]:3d}  {k}")
PY
