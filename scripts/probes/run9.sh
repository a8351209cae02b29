timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 900 python scripts/probes/precision_probe.py > gpurun_out/prec_final.txt 2>&1; tail -1 gpurun_out/prec_final.txt
