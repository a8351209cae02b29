# A/B (alternating, same box): backward-weight per call at a few C5 rows, in-tree vs $1
for s in 256,256,2,50%,32,14,14 512,512,8,50%,32,14,14 256,256,2,50%,32,56,56 1024,1024,4,25%,32,56,56; do
  for i in 1 2; do
    echo "cur $s: $(SCC_SHAPE=$s OPS=bwt timeout 120 python scripts/probes/small_ops.py 2>&1 | tail -1)"
    echo "alt $s: $(SCC_SHAPE=$s OPS=bwt SCC_LIB_PATH=$1/libscc_b200.so timeout 120 python scripts/probes/small_ops.py 2>&1 | tail -1)"
  done
done
