"""Run every SCC layer shape of SCC-ResNet-18 / SCC-VGG16 (batch 128) through
forward / backward-data / backward-weight and check against a dense torch fp32
reference of the same operator (masked 1x1 conv)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2101_00745_b200 as scc
from paper_2101_00745_b200 import _lib
shapes = [(64, 64, 32), (64, 128, 16), (128, 128, 16), (128, 256, 8), (256, 256, 8), (256, 512, 4), (512, 512, 4),
          (128, 128, 32), (256, 256, 16), (512, 512, 8), (512, 512, 2)]
def dense_w(cfg, w):
    ci, co, gw = cfg.c_in, cfg.c_out, cfg.group_width
    full = torch.zeros(co, ci, device=w.device, dtype=torch.float64)
    for oc in range(co):
        st = (oc * cfg.shift) % ci
        for s in range(gw):
            full[oc, (st + s) % ci] += w[oc * gw + s].double()
    return full
for ci, co, hw in shapes:
    for path in (_lib.SCC_PATH_AUTO, _lib.SCC_PATH_CUDA_CORE):
        cfg = scc.scc_config_new(ci, co, 2, "50%", True); cfg.set_path(path)
        n = 16
        x = torch.randn(n, ci, hw, hw, device="cuda"); gy = torch.randn(n, co, hw, hw, device="cuda")
        wts = scc.scc_weights_init(cfg); wts.bias.uniform_(-0.5, 0.5)
        try:
            y = scc.scc_forward(x, wts, cfg); g = scc.scc_backward(gy, x, wts, cfg)
            torch.cuda.synchronize()
        except Exception as ex:
            print(f"{ci}->{co} {hw}x{hw} path {path}: ERROR {ex}", flush=True); continue
        W = dense_w(cfg, wts.weight)
        yr = torch.einsum("oc,nchw->nohw", W, x.double()) + wts.bias.double().view(1, -1, 1, 1)
        dxr = torch.einsum("oc,nohw->nchw", W, gy.double())
        dWd = torch.einsum("nohw,nchw->oc", gy.double(), x.double())
        dwr = torch.stack([dWd[oc, [(((oc * cfg.shift) % ci) + s) % ci for s in range(cfg.group_width)]] for oc in range(co)]).reshape(-1)
        dbr = gy.double().sum((0, 2, 3))
        e = lambda a, b: float((a.double() - b).abs().max() / b.abs().max())
        print(f"{ci}->{co} {hw}x{hw} path {cfg.path_for(n, hw, hw)}: fwd {e(y, yr):.1e} dx {e(g.grad_input, dxr):.1e} dw {e(g.params.grad_weight, dwr):.1e} db {e(g.params.grad_bias, dbr):.1e}", flush=True)
