"""Measured norm-relative errors (max|d|/max|ref|, the reference's metric) of
every C5 shape at its full batch (N=32) on the tensor-core path against the
fp64 reference (tests/fp64_ref.py): y, dx, dW, db.  Run with the default
build (3xTF32 forward, bf16x3 backward) or with a -DSCC_FWD_BF16 build loaded
through SCC_LIB_PATH (bf16x3 forward on the generation-1 kernels)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tests"))
import torch
import paper_2101_00745_b200 as scc
from paper_2101_00745_b200 import _lib
from fp64_ref import scc_fp64
def nrel(a, b):
    return float((a.double() - b).abs().max() / b.abs().max().clamp_min(1e-300))
worst = {}
for c in (256, 512, 1024):
    for hw in (56, 14):
        for cg in (2, 4, 8):
            for co in ("25%", "50%", "75%"):
                cfg = scc.scc_config_new(c, c, cg, co, True)
                gen = torch.Generator(device="cuda").manual_seed(1)
                x = torch.randn(32, c, hw, hw, device="cuda", generator=gen)
                dy = torch.randn(32, c, hw, hw, device="cuda", generator=gen)
                wts = scc.scc_weights_init(cfg)
                wts.bias.uniform_(-0.5, 0.5)
                ry, rdx, rdw, rdb = scc_fp64(c, c, cfg.group_width, cfg.shift, x, wts.weight, wts.bias, dy)
                cfg.set_path(_lib.SCC_PATH_TENSOR)
                y = scc.scc_forward(x, wts, cfg)
                g = scc.scc_backward(dy, x, wts, cfg)
                e = {"y": nrel(y, ry), "dx": nrel(g.grad_input, rdx), "dw": nrel(g.params.grad_weight, rdw),
                     "db": nrel(g.params.grad_bias, rdb)}
                for k, v in e.items():
                    worst[k] = max(worst.get(k, 0.0), v)
                print(json.dumps({"C": c, "hw": hw, "cg": cg, "co": co, **{k: float(f"{v:.3e}") for k, v in e.items()}}), flush=True)
                del x, dy, ry, rdx, rdw, rdb, y, g
                torch.cuda.empty_cache()
print(json.dumps({"worst": {k: float(f"{v:.3e}") for k, v in worst.items()}}))
