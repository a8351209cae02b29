#!/bin/bash
# One kernel iteration: parity subset, timing, optional ncu capture of $1 (kernel regex).
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_scc_gpu.py -q -x -k "not sweep_full_size_properties" > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 120 python scripts/bwd_timing.py 2>&1 | head -3
if [ -n "$1" ]; then
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"$1" -s 3 -c 1 -o gpurun_out/prof_iter -f python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-models --no-graph --no-traffic > /dev/null 2>&1; ls -la gpurun_out/prof_iter.ncu-rep
fi
