#!/bin/bash
# quick loop: forward / backward-data (gen 2) parity + timeline, A/B of the epilogue store mode
mkdir -p gpurun_out
if [ "$1" != "notest" ]; then timeout 600 python -m pytest tests/test_scc_gpu.py -m gpu -x -q > gpurun_out/quick_tests.log 2>&1; tail -1 gpurun_out/quick_tests.log; fi
make -s -C paper_2101_00745_b200/csrc SCC_EXTRA=-DSCC_TRACE OUT=/tmp/tr -j8 > /dev/null 2>&1
SCC_LIB_PATH=/tmp/tr/libscc_b200.so timeout 120 python scripts/band_timing.py 32 64 128 32 32 2 x 2>&1 | grep -v "grp1\|MHz"
echo "--- 32-row group stores"
SCC_FWD_R32=1 SCC_LIB_PATH=/tmp/tr/libscc_b200.so timeout 120 python scripts/band_timing.py 32 64 128 32 32 2 x 2>&1 | grep -v "grp1\|MHz"
