#!/bin/bash
# One measurement round: bench line, reference arm, launch list, full ncu
# capture of the top kernel.  Outputs under gpurun_out/.
mkdir -p gpurun_out
timeout 300 python bench.py --steps 200 --warmup 10 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -1 gpurun_out/bench.json | cut -c1-400
timeout 300 python bench.py --impl reference --steps 10 --warmup 1 > gpurun_out/bench_ref.json 2>&1; tail -1 gpurun_out/bench_ref.json | cut -c1-300
scripts/ncu_launches.sh gpurun_out/launches.csv --no-graph > gpurun_out/launches.txt 2>&1; cat gpurun_out/launches.txt
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"${1:-tc_weight_kernel}" -s 3 -c 1 -o gpurun_out/prof_top python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-models --no-graph > /dev/null 2>&1; ls -la gpurun_out/prof_top.ncu-rep
