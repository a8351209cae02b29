"""Run the fused DW3x3+SCC forward (scc_dsc_forward_t_f32), the plain SCC
forward and the one-pass depthwise backward a few times at
$DSC_SHAPE ("ci,co,n,hw", default 64,64,128,32) for ncu captures."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2101_00745_b200 as scc
ci, co, n, hw = (int(v) for v in os.environ.get("DSC_SHAPE", "64,64,128,32").split(","))
cfg = scc.scc_config_new(ci, co, 2, "50%", False)
x = torch.randn(n, ci, hw, hw, device="cuda")
dw = torch.randn(ci, 1, 3, 3, device="cuda") / 3
wts = scc.scc_weights_init(cfg)
gy = torch.randn_like(x)
for _ in range(4):
    y, t = scc.dsc_forward_t(x, dw, None, wts, cfg, 1)
    y2 = scc.scc_forward(t, wts, cfg)
    dx, ddw, _ = scc.dw3x3_backward(gy, x, dw, 1)
torch.cuda.synchronize()
print("ok")
