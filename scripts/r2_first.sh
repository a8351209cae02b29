set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 300 python bench.py --steps 50 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -1 gpurun_out/bench.json | cut -c1-600
make -s -C paper_2101_00745_b200/csrc SCC_EXTRA=-DSCC_TRACE OUT=/tmp/tr -j8 > /dev/null 2>&1
SCC_LIB_PATH=/tmp/tr/libscc_b200.so timeout 120 python scripts/bwd_timing.py > gpurun_out/bwd_timing.txt 2>&1; cat gpurun_out/bwd_timing.txt
