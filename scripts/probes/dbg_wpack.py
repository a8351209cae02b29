import sys, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2101_00745_b200 as scc
from fp64_ref import scc_fp64
from test_scc_gpu import _nrel_t
for (ci, co, cg, ov, n, h, w) in [(512, 512, 2, "50%", 1, 4, 4), (512, 512, 2, "50%", 4, 4, 4), (256, 256, 2, "50%", 13, 4, 4),
                                  (1024, 1024, 2, "75%", 1, 2, 2), (256, 256, 2, "50%", 8, 2, 4), (256, 256, 2, "50%", 8, 8, 8)]:
    for path in (2, 3):
        cfg = scc.scc_config_new(ci, co, cg, ov, True); cfg.set_path(path)
        x = torch.randn(n, ci, h, w, device="cuda"); dy = torch.randn(n, co, h, w, device="cuda")
        wts = scc.scc_weights_init(cfg)
        ry, rdx, rdw, rdb = scc_fp64(ci, co, cfg.group_width, cfg.shift, x, wts.weight, wts.bias, dy)
        pg = scc.scc_backward_params(dy, x, cfg); torch.cuda.synchronize()
        dw = pg.grad_weight.double()
        print((ci, co, n, h, w), "path", path, f"dw err {_nrel_t(pg.grad_weight, rdw):.2e} db err {_nrel_t(pg.grad_bias, rdb):.2e}",
              f"|dw| {dw.abs().max().item():.3g} |ref| {rdw.abs().max().item():.3g} ratio-fit {(dw * rdw).sum().item() / (rdw * rdw).sum().item():.3f}", flush=True)
