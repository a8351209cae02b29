#!/bin/bash
# Fused-backward iteration: parity (scc + models), timeline, bench, host sweep.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_scc_gpu.py tests/test_models.py tests/test_refharness.py tests/test_cpp_shim.py -q -x > gpurun_out/gpu_tests.log 2>&1; tail -15 gpurun_out/gpu_tests.log
make -s -C paper_2101_00745_b200/csrc SCC_EXTRA=-DSCC_TRACE OUT=/tmp/tr -j8 > /dev/null 2>&1
SCC_LIB_PATH=/tmp/tr/libscc_b200.so timeout 120 python scripts/bwd_timing.py > gpurun_out/bwd_timing.txt 2>&1; cat gpurun_out/bwd_timing.txt
timeout 600 python bench.py --steps 50 --warmup 5 --no-models > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -1 gpurun_out/bench.json | cut -c1-2500; tail -3 gpurun_out/bench.err
timeout 600 python scripts/host_sweep.py > gpurun_out/host_sweep.txt 2>&1; cat gpurun_out/host_sweep.txt
