timeout 600 python -m pytest tests/test_scc_gpu.py -m gpu -x -q 2>&1 | tail -2
bash scripts/probes/ab_bwd.sh
make -s -C paper_2101_00745_b200/csrc SCC_EXTRA=-DSCC_TRACE OUT=/tmp/tr -j8 > /dev/null 2>&1
SCC_LIB_PATH=/tmp/tr/libscc_b200.so timeout 120 python scripts/bwd_timing.py 2>&1 | grep -v "^raw" | tail -2 | cut -c1-400
