#!/bin/bash
for rep in 1 2 3; do
  for lib in new old; do
    if [ $lib = old ]; then export SCC_LIB_PATH=$PWD/scripts/probes/_ab/libscc_b200.so; else unset SCC_LIB_PATH; fi
    echo "$lib $(SCC_SHAPE=1024,1024,8,50%,32,56,56 OPS=bdata,fwd timeout 120 python scripts/probes/small_ops.py | tr '\n' ' ')"
  done
done
