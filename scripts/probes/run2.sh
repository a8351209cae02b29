mkdir -p gpurun_out

timeout 600 python -m pytest tests/test_scc_gpu.py -m gpu -x -q > gpurun_out/quick_tests.log 2>&1; tail -30 gpurun_out/quick_tests.log
timeout 120 python scripts/bwd_timing.py 2>&1 | head -5
make -s -C paper_2101_00745_b200/csrc SCC_EXTRA=-DSCC_TRACE OUT=/tmp/tr -j8 > /dev/null 2>&1
SCC_LIB_PATH=/tmp/tr/libscc_b200.so timeout 120 python scripts/bwd_timing.py 2>&1 | grep -v "^raw"
