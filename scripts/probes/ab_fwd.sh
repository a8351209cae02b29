# A/B (alternating, same box) of the c1 forward: in-tree library vs $1
for i in 1 2 3; do
  echo "cur:  $(timeout 120 python scripts/band_timing.py 32 64 128 32 32 2 x 2>&1 | head -2 | tr '\n' ' ')"
  echo "alt:  $(SCC_LIB_PATH=$1/libscc_b200.so timeout 120 python scripts/band_timing.py 32 64 128 32 32 2 x 2>&1 | head -2 | tr '\n' ' ')"
done
