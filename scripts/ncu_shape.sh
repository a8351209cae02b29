#!/bin/bash
# Full ncu capture of one kernel of one op at one shape (eager calls of
# scripts/probes/small_ops.py).
# Usage: scripts/ncu_shape.sh SHAPE(ci,co,cg,ov%,n,h,w) OP(fwd|bdata|bwt) KERNEL_REGEX OUT
SCC_SHAPE=$1 OPS=$2 EAGER=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$3" -s 2 -c 1 \
  -o "$4" -f python scripts/probes/small_ops.py > /dev/null 2>&1
ls -la "$4.ncu-rep"
