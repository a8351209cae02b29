#!/bin/bash
make -s -C paper_2101_00745_b200/csrc SCC_EXTRA=-DSCC_TRACE OUT=/tmp/tr -j8 > /dev/null 2>&1
SCC_LIB_PATH=/tmp/tr/libscc_b200.so timeout 120 python scripts/band_timing.py 32 64 128 32 32 2 x 2>&1
SCC_LIB_PATH=/tmp/tr/libscc_b200.so timeout 120 python scripts/bwd_timing.py 2>&1
