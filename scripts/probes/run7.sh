make -s -C paper_2101_00745_b200/csrc SCC_EXTRA=-DSCC_TRACE OUT=/tmp/tr -j8 > /dev/null 2>&1
SCC_LIB_PATH=/tmp/tr/libscc_b200.so timeout 120 python scripts/band_timing.py 32 64 128 32 32 2 x 2>&1 | tail -12
timeout 300 python bench.py --steps 100 --warmup 10 --no-models --no-compositions > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; tail -1 gpurun_out/bench_q.json | cut -c1-1500
