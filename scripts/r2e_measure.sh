#!/bin/bash
# Round-2 (final) measurement: GPU tests, bench line (+ reference arm),
# launch list, full ncu captures of the c1 fused backward / forward and of the
# generation-1 bf16x3 backward kernels at a C5 shape, the dsc_block kernels
# (fused DW+SCC forward, one-pass depthwise backward), full C5 sweep.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -1 gpurun_out/gpu_tests.log
timeout 900 python bench.py --steps 200 --warmup 10 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -1 gpurun_out/bench.json | cut -c1-300
timeout 300 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/bench_ref.json 2>&1; tail -1 gpurun_out/bench_ref.json | cut -c1-300
scripts/ncu_launches.sh gpurun_out/launches.csv --no-graph --no-traffic --no-compositions > gpurun_out/launches.txt 2>&1; cat gpurun_out/launches.txt
for k in tc_bwd_kernel tc_band2_kernel; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 3 -c 1 -o gpurun_out/prof_$k -f \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-models --no-graph --no-traffic --no-compositions --no-c5 > /dev/null 2>&1
  ls gpurun_out/prof_$k.ncu-rep
done
S=256,256,2,50%,32,56,56
scripts/ncu_shape.sh $S bdata tc_band_kernel gpurun_out/prof56_tc_band_kernel_bwd
scripts/ncu_shape.sh $S bwt tc_weight_kernel gpurun_out/prof56_tc_weight_kernel
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_band2 -s 0 -c 1 -o gpurun_out/prof_dsc_fused -f python scripts/probes/dsc_one.py > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:dw_bwd_kernel -s 0 -c 1 -o gpurun_out/prof_dw_bwd -f python scripts/probes/dsc_one.py > /dev/null 2>&1
ls gpurun_out/prof_dsc_fused.ncu-rep gpurun_out/prof_dw_bwd.ncu-rep
timeout 600 python scripts/dsc_timing.py > gpurun_out/dsc_timing.jsonl 2>&1
timeout 1200 python scripts/sweep.py --parts --out gpurun_out/sweep.json > gpurun_out/sweep.log 2>&1; tail -1 gpurun_out/sweep.log
