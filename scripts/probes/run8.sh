timeout 900 python scripts/probes/precision_probe.py > gpurun_out/prec_default.txt 2>&1; tail -1 gpurun_out/prec_default.txt
make -s -C paper_2101_00745_b200/csrc SCC_EXTRA=-DSCC_FWD_BF16 OUT=/tmp/fb -j8 > /dev/null 2>&1
SCC_LIB_PATH=/tmp/fb/libscc_b200.so timeout 900 python scripts/probes/precision_probe.py > gpurun_out/prec_fwdbf16.txt 2>&1; tail -1 gpurun_out/prec_fwdbf16.txt
SCC_LIB_PATH=/tmp/fb/libscc_b200.so timeout 600 python scripts/sweep.py --parts --co 50 --out gpurun_out/sweep_fb.json > gpurun_out/sweep_fb.log 2>&1; tail -1 gpurun_out/sweep_fb.log
