#!/bin/bash
# Round-2 final profiles: launch list of the c1 step, full ncu captures of the
# c1 forward / fused backward and of the generation-1 kernels at C256 14x14 cg2.
mkdir -p gpurun_out
scripts/ncu_launches.sh gpurun_out/launches.csv --no-graph --no-traffic --no-compositions > gpurun_out/launches.txt 2>&1; cat gpurun_out/launches.txt
for k in tc_bwd_kernel tc_band2_kernel; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 3 -c 1 -o gpurun_out/prof_$k -f \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-models --no-graph --no-traffic --no-compositions --no-c5 > /dev/null 2>&1
  ls -la gpurun_out/prof_$k.ncu-rep
done
S=256,256,2,50%,32,14,14
scripts/ncu_shape.sh $S fwd tc_band_kernel gpurun_out/prof14_tc_band_kernel
scripts/ncu_shape.sh $S bwt tc_weight_kernel gpurun_out/prof14_tc_weight_kernel
scripts/ncu_shape.sh $S bwt tc_weight_finalize gpurun_out/prof14_tc_weight_finalize
