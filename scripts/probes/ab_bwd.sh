# A/B of the fused backward: in-tree library vs build/lib_prev (alternating, same box)
for i in 1 2 3; do
  echo "cur:  $(timeout 120 python scripts/bwd_timing.py 2>&1 | head -3 | tr '\n' ' ')"
  echo "prev: $(SCC_LIB_PATH=build/lib_prev/libscc_b200.so timeout 120 python scripts/bwd_timing.py 2>&1 | head -3 | tr '\n' ' ')"
done
