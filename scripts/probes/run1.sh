mkdir -p gpurun_out
timeout 120 python scripts/probes/bf16_probe.py > gpurun_out/bf16_probe.txt 2>&1; cat gpurun_out/bf16_probe.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 200 --warmup 10 --no-models > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -1 gpurun_out/bench.json | cut -c1-700
