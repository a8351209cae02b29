timeout 900 python -m pytest tests/test_scc_gpu.py -m gpu -x -q 2>&1 | tail -2
timeout 600 python scripts/sweep.py --parts --C 512 1024 --cg 2 4 --co 25 75 --out gpurun_out/sweep_nc.json > gpurun_out/sweep_nc.log 2>&1; grep '"C"' gpurun_out/sweep_nc.log | python -c "
import sys, json
for l in sys.stdin:
    r = json.loads(l); print(r['C'], r['hw'], r['cg'], r['co'], 'bw', r['us']['bwd_weight'], 'step', r['us']['step'], 'frac', r['hbm_frac_step'])
"
