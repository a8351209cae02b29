make -s -C paper_2101_00745_b200/csrc SCC_EXTRA=-DSCC_TRACE OUT=/tmp/tr -j8 > /dev/null 2>&1
for s in 1024,1024,2,50%,32,56,56 256,256,2,50%,32,56,56; do
  for op in bdata fwd; do
    echo "$s $op: $(SCC_SHAPE=$s OP=$op SCC_LIB_PATH=/tmp/tr/libscc_b200.so timeout 120 python scripts/band1_timeline.py 2>&1 | tail -1)"
  done
done
