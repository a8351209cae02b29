#!/bin/bash
# Watchdog-build smoke of the tensor-core kernels: any mbarrier wait that
# would hang is cut short and counted instead.
export SCC_LIB_PATH=build/wd/libscc_wd.so
timeout 100 python scripts/hang_probe.py 2>&1 | tail -3
timeout 60 python scripts/hang_probe_w.py 2>&1 | tail -1
timeout 200 python -m pytest tests/test_scc_gpu.py -x -q -k "tensor" 2>&1 | tail -4
