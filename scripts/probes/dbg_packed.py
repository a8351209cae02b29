import sys, os, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2101_00745_b200 as scc
from paper_2101_00745_b200 import _lib
from fp64_ref import scc_fp64
from test_scc_gpu import _nrel_t
for (ci, co, cg, ov, n, h, w) in [(96, 96, 3, "50%", 3, 4, 8), (96, 96, 3, "50%", 4, 4, 8), (96, 96, 3, "50%", 3, 8, 16), (64, 64, 2, "50%", 3, 4, 8)]:
    for path in (2, 3):
        cfg = scc.scc_config_new(ci, co, cg, ov, True); cfg.set_path(path)
        x = torch.randn(n, ci, h, w, device="cuda"); dy = torch.randn(n, co, h, w, device="cuda")
        wts = scc.scc_weights_init(cfg)
        ry, rdx, rdw, rdb = scc_fp64(ci, co, cfg.group_width, cfg.shift, x, wts.weight, wts.bias, dy)
        dx = scc.scc_backward_input(dy, wts, cfg); torch.cuda.synchronize()
        e = _nrel_t(dx, rdx)
        bad = (dx.double() - rdx).abs().amax(dim=(2, 3)) > 1e-3
        print((ci, co, n, h, w), "path", path, "dx err", f"{e:.2e}", "bad (n,c):", bad.nonzero()[:6].tolist(), flush=True)
