#!/bin/bash
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:tc_band2 -s 2 -c 2 -o gpurun_out/dsc_fused -f python scripts/probes/dsc_one.py > gpurun_out/dsc_ncu.log 2>&1
tail -3 gpurun_out/dsc_ncu.log
