make -s -C paper_2101_00745_b200/csrc SCC_EXTRA=-DSCC_TRACE OUT=/tmp/tr -j8 > /dev/null 2>&1
CTA_DUMP=1 SCC_LIB_PATH=/tmp/tr/libscc_b200.so timeout 120 python scripts/bwd_timing.py 2>&1 | grep -v "^raw" > gpurun_out/cta_dump.txt; tail -3 gpurun_out/cta_dump.txt
