#!/bin/bash
# depthwise backward: the two separate kernels vs scc_dw3x3_backward_f32
python scripts/dsc_timing.py 2>&1 | tee gpurun_out/dsc_t.jsonl | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print(' ', d['c_in'], d['hw'], d['stride'], 'sep', round(d['dw_bwd_data_ours_us'] + d['dw_bwd_weight_ours_us'], 2), 'one', d['dw_bwd_ours_us'], 'fwd fused', d['fused_t_us'], 'pair', d['pair_ours_us'])
"
