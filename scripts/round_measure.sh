#!/bin/bash
# One measurement round: GPU tests, bench line, reference arm, launch list,
# full ncu capture of the step's dominant kernel, C5 sweep.  Outputs under
# gpurun_out/.  Usage: scripts/round_measure.sh [KERNEL_REGEX]
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -1 gpurun_out/gpu_tests.log
timeout 300 python bench.py --steps 200 --warmup 10 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -1 gpurun_out/bench.json | cut -c1-400
timeout 300 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/bench_ref.json 2>&1; tail -1 gpurun_out/bench_ref.json | cut -c1-300
scripts/ncu_launches.sh gpurun_out/launches.csv --no-graph > gpurun_out/launches.txt 2>&1; cat gpurun_out/launches.txt
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"${1:-tc_bwd_kernel}" -s 3 -c 1 -o gpurun_out/prof_top python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-models --no-graph > /dev/null 2>&1; ls -la gpurun_out/prof_top.ncu-rep
timeout 600 python scripts/sweep.py --parts --out gpurun_out/sweep.json > gpurun_out/sweep.log 2>&1; tail -1 gpurun_out/sweep.log
