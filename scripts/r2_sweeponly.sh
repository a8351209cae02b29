#!/bin/bash
mkdir -p gpurun_out
timeout 900 python scripts/sweep.py --parts --out gpurun_out/sweep.json > gpurun_out/sweep.log 2>&1; tail -1 gpurun_out/sweep.log
