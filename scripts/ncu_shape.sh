#!/bin/bash
# Full ncu capture of one kernel of one op at one shape.
# Usage: scripts/ncu_shape.sh SHAPE(ci,co,cg,ov%,n,h,w) OP KERNEL_REGEX OUT
SCC_SHAPE=$1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$3" -s 2 -c 1 \
  -o "$4" python scripts/one_op.py "$2" > /dev/null 2>&1
ls -la "$4.ncu-rep"
