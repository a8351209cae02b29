"""The composition baselines (paper_2101_00745_b200/compose.py: the paper's
"Base" SCC from stock operators) against the reference's composition routes
(reference.cpp:335-490, via oracle/_ref) on CPU in fp64, and against the SCC
kernels on the GPU in fp32."""
import numpy as np
import pytest
import torch

from conftest import norm_rel

GEOMS = [(8, 16, 4, "50%"), (6, 4, 2, "1"), (12, 12, 3, "2"), (16, 24, 4, "25%"), (8, 5, 4, "1"), (6, 6, 1, "0")]


def _cfgs(ref, ci, co, cg, ov):
    import paper_2101_00745_b200 as scc
    cfg = scc.scc_config_new(ci, co, cg, ov, True)
    ovl = ("ratio", float(ov[:-1]) / 100) if ov.endswith("%") else ("channels", int(ov))
    return cfg, ref.config(ci, co, cg, ovl, True)


@pytest.mark.parametrize("route", ["channel", "conv"])
@pytest.mark.parametrize("use_cc", [False, True])
def test_compose_matches_reference_fp64(ref, route, use_cc):
    from paper_2101_00745_b200 import compose
    rng = np.random.default_rng(7)
    for ci, co, cg, ov in GEOMS:
        cfg, rc = _cfgs(ref, ci, co, cg, ov)
        x = rng.standard_normal((2, ci, 3, 4))
        w = rng.standard_normal(co * cfg.group_width)
        b = rng.standard_normal(co)
        dy = rng.standard_normal((2, co, 3, 4))
        t = lambda a: torch.from_numpy(a)  # noqa: E731
        y, aux = compose.ROUTES[route](t(x), t(w), t(b), cfg, use_cc)
        ry, raux = ref.compose_forward(rc, route, use_cc, x, w, b)
        assert aux == raux
        assert norm_rel(y.numpy(), ry) <= 1e-12
        dx, dw, db = compose.compose_backward(route, use_cc, t(dy), t(x), t(w), t(b), cfg)
        rdx, rdw, rdb = ref.compose_backward(rc, route, use_cc, dy, x, w)
        assert norm_rel(dx.numpy(), rdx) <= 1e-12
        assert norm_rel(dw.numpy(), rdw) <= 1e-12
        assert norm_rel(db.numpy(), rdb) <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("route", ["channel", "conv"])
def test_compose_gpu_matches_scc_kernels(route):
    """fp32 on the B200 (TF32 off): the Base routes and the SCC kernels agree
    within the parity bars at config 1's geometry."""
    import paper_2101_00745_b200 as scc
    from paper_2101_00745_b200 import compose
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False
    cfg = scc.scc_config_new(64, 128, 2, "50%", True)
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(4, 64, 16, 16, device="cuda", generator=g)
    dy = torch.randn(4, 128, 16, 16, device="cuda", generator=g)
    wts = scc.scc_weights_init(cfg)
    wts.bias.uniform_(-0.5, 0.5)
    y = scc.scc_forward(x, wts, cfg)
    gr = scc.scc_backward(dy, x, wts, cfg)
    for use_cc in (False, True):
        yc, _ = compose.ROUTES[route](x, wts.weight, wts.bias, cfg, use_cc)
        assert norm_rel(yc.cpu().numpy(), y.cpu().numpy()) <= 1e-5
        dx, dw, db = compose.compose_backward(route, use_cc, dy, x, wts.weight, wts.bias, cfg)
        assert norm_rel(dx.cpu().numpy(), gr.grad_input.cpu().numpy()) <= 1e-4
        assert norm_rel(dw.cpu().numpy(), gr.params.grad_weight.cpu().numpy()) <= 1e-4
        assert norm_rel(db.cpu().numpy(), gr.params.grad_bias.cpu().numpy()) <= 1e-4
