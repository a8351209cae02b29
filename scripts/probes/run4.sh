mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_bwd_kernel -s 5 -c 1 -o gpurun_out/bwd_full -f python scripts/bwd_timing.py > /dev/null 2>&1
ncu -i gpurun_out/bwd_full.ncu-rep --page source --csv > gpurun_out/bwd_source.csv 2>&1
ncu -i gpurun_out/bwd_full.ncu-rep --page details --csv > gpurun_out/bwd_details.csv 2>&1
ls -la gpurun_out/
