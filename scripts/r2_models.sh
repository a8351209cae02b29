#!/bin/bash
mkdir -p gpurun_out
timeout 900 python scripts/model_bench.py > gpurun_out/models.jsonl 2> gpurun_out/models.err; cat gpurun_out/models.jsonl; tail -3 gpurun_out/models.err
for m in resnet18 resnet50; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof_$m.csv python scripts/model_profile.py $m > /dev/null 2>&1
python - gpurun_out/prof_$m.csv <<'PY'
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[0].isdigit()]
agg = collections.Counter(); tot = 0
for r in rows:
    v = float(r[-1].replace(",", "")); tot += v
    n = r[4]
    k = ("scc:" + n.split("(")[0].split("::")[-1][:40]) if "scc::" in n else ("torch:" + n.split("(")[0][-50:])
    agg[k] += v
print(f"total {tot/1e3:.1f} us over {len(rows)} kernels (cold, serialised)")
for k, v in agg.most_common(25): print(f"{v/1e3:10.1f} us {100*v/tot:5.1f}%  {k}")
PY
done
