# A/B (alternating, same box): in-tree library vs build/lib_prev -- fused backward and c1 forward
for i in 1 2 3; do
  echo "cur:  $(timeout 120 python scripts/bwd_timing.py 2>&1 | head -3 | tr '\n' ' ') $(timeout 120 python scripts/band_timing.py 32 64 128 32 32 2 x 2>&1 | head -1)"
  echo "prev: $(SCC_LIB_PATH=build/lib_prev/libscc_b200.so timeout 120 python scripts/bwd_timing.py 2>&1 | head -3 | tr '\n' ' ') $(SCC_LIB_PATH=build/lib_prev/libscc_b200.so timeout 120 python scripts/band_timing.py 32 64 128 32 32 2 x 2>&1 | head -1)"
done
