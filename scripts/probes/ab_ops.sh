# A/B (alternating, same box) of one op ($2: fwd|bdata|bwt) at C5 rows: in-tree vs $1
for s in 1024,1024,2,50%,32,56,56 1024,1024,4,50%,32,56,56 512,512,2,50%,32,56,56 256,256,2,50%,32,56,56 1024,1024,2,50%,32,14,14; do
  for i in 1 2; do
    echo "cur $s: $(SCC_SHAPE=$s OPS=$2 timeout 120 python scripts/probes/small_ops.py 2>&1 | tail -1)"
    echo "alt $s: $(SCC_SHAPE=$s OPS=$2 SCC_LIB_PATH=$1/libscc_b200.so timeout 120 python scripts/probes/small_ops.py 2>&1 | tail -1)"
  done
done
