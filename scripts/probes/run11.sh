echo "--- with the chain cap"; timeout 900 python scripts/probes/chain_probe.py 2>&1 | tail -7
echo "--- before"; SCC_LIB_PATH=build/lib_prev/libscc_b200.so timeout 900 python scripts/probes/chain_probe.py 2>&1 | tail -7
