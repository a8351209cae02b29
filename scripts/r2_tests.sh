#!/bin/bash
# GPU test pass + a short bench (with the in-run traffic pass) + host pipeline sweep.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --durations=20 > gpurun_out/gpu_tests.log 2>&1; tail -40 gpurun_out/gpu_tests.log
timeout 600 python scripts/host_sweep.py > gpurun_out/host_sweep.txt 2>&1; cat gpurun_out/host_sweep.txt
timeout 600 python bench.py --steps 50 --warmup 5 --no-models > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -1 gpurun_out/bench.json | cut -c1-3000
