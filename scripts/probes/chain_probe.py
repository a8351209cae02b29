"""dW error vs the accumulation-chain length of the generation-1 backward-weight
split partials: C=1024 / 512 cg=2 at 14x14 for growing N (tensor path, fp64
reference), current library vs SCC_LIB_PATH."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tests"))
import torch
import paper_2101_00745_b200 as scc
from paper_2101_00745_b200 import _lib
from fp64_ref import scc_fp64
def nrel(a, b):
    return float((a.double() - b).abs().max() / b.abs().max())
for c, hw, n in ((512, 14, 32), (512, 14, 256), (512, 14, 1024), (1024, 14, 32), (1024, 14, 512), (1024, 56, 32), (1024, 56, 96)):
    cfg = scc.scc_config_new(c, c, 2, "50%", True)
    gen = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn(n, c, hw, hw, device="cuda", generator=gen)
    dy = torch.randn(n, c, hw, hw, device="cuda", generator=gen)
    wts = scc.scc_weights_init(cfg)
    _, _, rdw, rdb = scc_fp64(c, c, cfg.group_width, cfg.shift, x, wts.weight, wts.bias, dy)
    cfg.set_path(_lib.SCC_PATH_TENSOR)
    pg = scc.scc_backward_params(dy, x, cfg)
    torch.cuda.synchronize()
    print(f"C={c} {hw}x{hw} N={n}: dW {nrel(pg.grad_weight, rdw):.2e} db {nrel(pg.grad_bias, rdb):.2e}", flush=True)
    del x, dy, rdw, rdb, pg
    torch.cuda.empty_cache()
