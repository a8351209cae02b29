#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 900 python scripts/sweep.py --parts --out gpurun_out/sweep.json > gpurun_out/sweep.log 2>&1; tail -60 gpurun_out/sweep.log
