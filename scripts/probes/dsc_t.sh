#!/bin/bash
# fused DW3x3+SCC tensor-core forward: parity tests, then timing vs the pair
mkdir -p gpurun_out
python -m pytest tests/test_dsc_gpu.py -q 2>&1 | tail -15
python scripts/dsc_timing.py 2>&1 | tee gpurun_out/dsc_t.jsonl | tail -10
