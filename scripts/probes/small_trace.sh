#!/bin/bash
# gen-1 band kernel timeline (forward) at 14x14 sweep shapes, trace build
make -s -C paper_2101_00745_b200/csrc SCC_EXTRA=-DSCC_TRACE OUT=/tmp/tr -j8 > /dev/null 2>&1
for s in 256,256,2,50%,32,14,14 256,256,8,50%,32,14,14 512,512,4,50%,32,14,14 1024,1024,8,50%,32,14,14; do
  echo "== $s"
  SCC_SHAPE=$s SCC_LIB_PATH=/tmp/tr/libscc_b200.so timeout 60 python scripts/band1_timeline.py 2>&1 | tail -2
done
