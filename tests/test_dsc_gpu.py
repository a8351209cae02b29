"""Fused dsc_block (model.cpp:213-220: depthwise 3x3 then SCC) on the B200.

Forward: scc_dsc_forward_f32 against the CPU oracle composition
port.dw_forward (restating reference.cpp:74-123, pinned to the compiled
reference in test_oracle.py) -> port.forward (kernel.cpp:29-69), fp64 on the
same fp32 inputs, norm-relative <= 1e-5.  Backward: the depthwise kernels and
the whole DSC2d composition against the compiled reference's own
grouped_conv_backward (reference.cpp:155-247, via oracle/ref_shim.cpp) and
scc_backward_input / scc_backward_params (kernel.cpp:98-181), <= 1e-4; plus
float64 torch autograd of the same composition as a second check."""
import numpy as np
import pytest

from conftest import norm_rel

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

FWD_TOL = 1e-5
GRAD_TOL = 1e-4

CASES = [  # c_in, c_out, cg, co, n, h, w, stride, dw_bias, bias
    (64, 128, 2, "50%", 2, 8, 8, 1, False, True),
    (64, 128, 2, "50%", 3, 9, 9, 2, True, True),
    (48, 80, 3, 1, 2, 7, 5, 1, True, False),
    (32, 32, 4, "25%", 1, 1, 1, 1, False, True),
    (16, 24, 2, "75%", 2, 6, 6, 2, False, False),
    (128, 256, 2, "50%", 2, 16, 16, 2, False, True),
]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def _problem(case, seed=0):
    ci, co, cg, ov, n, h, w, s, dwb, hb = case
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n, ci, h, w)).astype(np.float32)
    dww = rng.uniform(-1 / 3, 1 / 3, (ci, 3, 3)).astype(np.float32)
    dwbias = rng.uniform(-0.5, 0.5, ci).astype(np.float32) if dwb else None
    return x, dww, dwbias


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}-{c[1]}-cg{c[2]}-{c[3]}-{c[5]}x{c[6]}-s{c[7]}")
def test_fused_forward_matches_oracle(port, case):
    import paper_2101_00745_b200 as scc
    ci, co, cg, ov, n, h, w, s, dwb, hb = case
    cfg = scc.scc_config_new(ci, co, cg, ov if isinstance(ov, str) else scc.Overlap.channels(ov), hb)
    x, dww, dwbias = _problem(case)
    rng = np.random.default_rng(1)
    gw = cfg.group_width
    wt = rng.uniform(-(1 / gw) ** 0.5, (1 / gw) ** 0.5, co * gw).astype(np.float32)
    b = rng.uniform(-0.5, 0.5, co).astype(np.float32) if hb else None
    wts = scc.SccWeights(torch.from_numpy(wt).cuda(), torch.from_numpy(b).cuda() if hb else None)
    y = scc.dsc_forward(torch.from_numpy(x).cuda(), torch.from_numpy(dww).cuda(),
                        torch.from_numpy(dwbias).cuda() if dwb else None, wts, cfg, s)
    t = port.dw_forward(x, dww, dwbias, 3, s)
    o = port.config(ci, co, cg, ("ratio", float(ov[:-1]) / 100) if isinstance(ov, str) else ("channels", ov), hb)
    ref = port.forward(o, t, wt, b)
    assert y.shape == ref.shape
    assert norm_rel(y.cpu().numpy(), ref) <= FWD_TOL
    y2 = scc.dsc_forward(torch.from_numpy(x).cuda(), torch.from_numpy(dww).cuda(),
                         torch.from_numpy(dwbias).cuda() if dwb else None, wts, cfg, s)
    assert torch.equal(y, y2)  # deterministic


@pytest.mark.parametrize("fused", [False, True], ids=["dw+scc", "fused"])
@pytest.mark.parametrize("case", [CASES[0], CASES[1], CASES[2]], ids=["s1", "s2-bias", "ragged"])
def test_dsc2d_autograd_matches_fp64(case, fused):
    import paper_2101_00745_b200 as scc
    ci, co, cg, ov, n, h, w, s, dwb, hb = case
    torch.manual_seed(0)
    layer = scc.DSC2d(ci, co, s, cg, ov if isinstance(ov, str) else scc.Overlap.channels(ov),
                      dw_bias=dwb, bias=hb, fused=fused, device="cuda")
    if hb:
        with torch.no_grad():
            layer.bias.uniform_(-0.5, 0.5)
    x = torch.randn(n, ci, h, w, device="cuda", requires_grad=True)
    y = layer(x)
    gy = torch.randn_like(y)
    y.backward(gy)
    cfg = layer.cfg
    # float64 reference: depthwise conv, then the SCC band as a dense 1x1 conv
    xd = x.detach().double().cpu().requires_grad_(True)
    dwd = layer.dw_weight.detach().double().cpu().requires_grad_(True)
    dbd = layer.dw_bias.detach().double().cpu().requires_grad_(True) if dwb else None
    wd = layer.weight.detach().double().cpu().requires_grad_(True)
    bd = layer.bias.detach().double().cpu().requires_grad_(True) if hb else None
    dense = torch.zeros(co, ci, dtype=torch.float64)
    rows, cols, slots = [], [], []
    for oc in range(co):
        st = (oc * cfg.shift) % ci
        for k in range(cfg.group_width):
            rows.append(oc); cols.append((st + k) % ci); slots.append(oc * cfg.group_width + k)
    dense = dense.index_put((torch.tensor(rows), torch.tensor(cols)), wd.reshape(-1)[torch.tensor(slots)])
    t = torch.nn.functional.conv2d(xd, dwd, dbd, s, 1, 1, ci)
    yd = torch.nn.functional.conv2d(t, dense.view(co, ci, 1, 1), bd)
    yd.backward(gy.double().cpu())
    assert norm_rel(y.detach().cpu().numpy(), yd.detach().numpy()) <= FWD_TOL
    assert norm_rel(x.grad.cpu().numpy(), xd.grad.numpy()) <= GRAD_TOL
    assert norm_rel(layer.dw_weight.grad.cpu().numpy(), dwd.grad.numpy()) <= GRAD_TOL
    assert norm_rel(layer.weight.grad.cpu().numpy(), wd.grad.numpy()) <= GRAD_TOL
    if dwb:
        assert norm_rel(layer.dw_bias.grad.cpu().numpy(), dbd.grad.numpy()) <= GRAD_TOL
    if hb:
        assert norm_rel(layer.bias.grad.cpu().numpy(), bd.grad.numpy()) <= GRAD_TOL


def test_dsc_argument_errors():
    import paper_2101_00745_b200 as scc
    cfg = scc.scc_config_new(8, 8, 2, "50%", True)
    wts = scc.scc_weights_init(cfg)
    x = torch.randn(1, 8, 4, 4, device="cuda")
    dww = torch.randn(8, 3, 3, device="cuda")
    with pytest.raises(scc.ArgumentError):
        scc.dsc_forward(x, dww, None, wts, cfg, 3)
    with pytest.raises(scc.ShapeError):
        scc.dsc_forward(x, dww[:4], None, wts, cfg, 1)
    with pytest.raises(scc.ShapeError):
        scc.dsc_forward(torch.randn(1, 4, 4, 4, device="cuda"), dww, None, wts, cfg, 1)


DW_SHAPES = [(2, 5, 7, 6, 1), (3, 4, 9, 9, 2), (1, 3, 1, 1, 1), (2, 8, 32, 32, 2), (1, 2, 112, 112, 1),
             (1, 2, 111, 113, 2)]


@pytest.mark.parametrize("shape", DW_SHAPES, ids=lambda s: f"{s[2]}x{s[3]}-s{s[4]}")
def test_dw3x3_forward_matches_oracle(port, shape):
    """The depthwise kernel against the C restatement of conv_forward_impl
    (pinned bit-exact to the compiled reference in test_oracle.py), including
    planes too large to stage in shared memory (112x112)."""
    import paper_2101_00745_b200 as scc
    n, c, h, w, s = shape
    rng = np.random.default_rng(5)
    x = rng.standard_normal((n, c, h, w)).astype(np.float32)
    wt = rng.uniform(-1 / 3, 1 / 3, (c, 3, 3)).astype(np.float32)
    b = rng.uniform(-0.5, 0.5, c).astype(np.float32)
    y = scc.dw3x3_forward(torch.from_numpy(x).cuda(), torch.from_numpy(wt).cuda(), torch.from_numpy(b).cuda(), s)
    assert norm_rel(y.cpu().numpy(), port.dw_forward(x, wt, b, 3, s)) <= FWD_TOL


@pytest.mark.parametrize("shape", DW_SHAPES, ids=lambda s: f"{s[2]}x{s[3]}-s{s[4]}")
def test_dw3x3_backward_matches_reference(ref, shape):
    """Depthwise backward-data / backward-weight / bias kernels against the
    reference's grouped_conv_backward (reference.cpp:155-247, groups = c)."""
    import paper_2101_00745_b200 as scc
    n, c, h, w, s = shape
    g = torch.Generator().manual_seed(3)
    x = torch.randn(n, c, h, w, generator=g)
    wt = torch.rand(c, 1, 3, 3, generator=g) - 0.5
    ho, wo = (h - 1) // s + 1, (w - 1) // s + 1
    gy = torch.randn(n, c, ho, wo, generator=g)
    rdx, rdw, rdb = ref.dw_backward(gy.numpy(), x.numpy(), wt.view(c, 3, 3).numpy(), 3, s, True)
    dx = scc.dw3x3_backward_data(gy.cuda(), wt.cuda(), (h, w), s)
    dw, db = scc.dw3x3_backward_weight(gy.cuda(), x.cuda(), s, True)
    assert norm_rel(dx.cpu().numpy(), rdx) <= GRAD_TOL
    assert norm_rel(dw.cpu().numpy(), rdw) <= GRAD_TOL
    assert norm_rel(db.cpu().numpy(), rdb) <= GRAD_TOL
    dw2, _ = scc.dw3x3_backward_weight(gy.cuda(), x.cuda(), s, True)
    assert torch.equal(dw, dw2)  # fixed-order reduction


@pytest.mark.parametrize("shape", DW_SHAPES + [(3, 64, 32, 32, 1), (2, 16, 7, 9, 1), (2, 16, 5, 6, 1)],
                         ids=lambda s: f"{s[1]}ch-{s[2]}x{s[3]}-s{s[4]}")
def test_dw3x3_backward_one_pass(ref, shape):
    """scc_dw3x3_backward_f32 (dx, dW, db from one pass over dy and x) against
    the reference's grouped_conv_backward; dx bitwise the separate
    backward-data kernel's (same per-element tap order), dW / db bitwise the
    separate weight kernel's on planes under 32 rows (same per-thread order;
    4-row blocks above that) and deterministic."""
    import paper_2101_00745_b200 as scc
    n, c, h, w, s = shape
    g = torch.Generator().manual_seed(6)
    x = torch.randn(n, c, h, w, generator=g)
    wt = torch.rand(c, 1, 3, 3, generator=g) - 0.5
    ho, wo = (h - 1) // s + 1, (w - 1) // s + 1
    gy = torch.randn(n, c, ho, wo, generator=g)
    rdx, rdw, rdb = ref.dw_backward(gy.numpy(), x.numpy(), wt.view(c, 3, 3).numpy(), 3, s, True)
    gyc, xc, wc = gy.cuda(), x.cuda(), wt.cuda()
    dx, dw, db = scc.dw3x3_backward(gyc, xc, wc, s, True)
    assert norm_rel(dx.cpu().numpy(), rdx) <= GRAD_TOL
    assert norm_rel(dw.cpu().numpy(), rdw) <= GRAD_TOL
    assert norm_rel(db.cpu().numpy(), rdb) <= GRAD_TOL
    sdx = scc.dw3x3_backward_data(gyc, wc, (h, w), s)
    sdw, sdb = scc.dw3x3_backward_weight(gyc, xc, s, True)
    assert torch.equal(dx, sdx)
    if h < 32 or s == 2:
        assert torch.equal(dw, sdw) and torch.equal(db, sdb)
    _, dw_nb, db_nb = scc.dw3x3_backward(gyc, xc, wc, s, False)
    assert db_nb is None and torch.equal(dw_nb, dw)


@pytest.mark.parametrize("fused", [False, True], ids=["dw+scc", "fused"])
@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}-{c[1]}-cg{c[2]}-{c[3]}-{c[5]}x{c[6]}-s{c[7]}")
def test_dsc2d_matches_reference_composition(ref, case, fused):
    """The whole dsc_block (model.cpp:213-220) forward and backward against
    the reference's own stages: grouped_conv_forward/_backward for the
    depthwise 3x3 and scc_forward / scc_backward_input / scc_backward_params."""
    import paper_2101_00745_b200 as scc
    ci, co, cg, ov, n, h, w, s, dwb, hb = case
    torch.manual_seed(1)
    layer = scc.DSC2d(ci, co, s, cg, ov if isinstance(ov, str) else scc.Overlap.channels(ov),
                      dw_bias=dwb, bias=hb, fused=fused, device="cuda")
    with torch.no_grad():
        if hb:
            layer.bias.uniform_(-0.5, 0.5)
        if dwb:
            layer.dw_bias.uniform_(-0.5, 0.5)
    x = torch.randn(n, ci, h, w, device="cuda", requires_grad=True)
    y = layer(x)
    gy = torch.randn_like(y)
    y.backward(gy)
    xn = x.detach().cpu().numpy()
    dww = layer.dw_weight.detach().cpu().numpy().reshape(ci, 3, 3)
    dwbn = layer.dw_bias.detach().cpu().numpy() if dwb else None
    wn = layer.weight.detach().cpu().numpy().reshape(-1)
    bn = layer.bias.detach().cpu().numpy() if hb else None
    o = ref.config(ci, co, cg, ov if isinstance(ov, str) else ("channels", ov), hb)
    t = ref.dw_forward(xn, dww, dwbn, 3, s)
    ry = ref.forward(o, t, wn, bn)
    gyn = gy.cpu().numpy()
    dt = ref.backward_input(o, gyn, wn)
    rdw, rdb = ref.backward_params(o, gyn, t)
    rdx, rddw, rddb = ref.dw_backward(dt, xn, dww, 3, s, dwb)
    assert norm_rel(y.detach().cpu().numpy(), ry) <= FWD_TOL
    assert norm_rel(x.grad.cpu().numpy(), rdx) <= GRAD_TOL
    assert norm_rel(layer.weight.grad.cpu().numpy().reshape(-1), rdw) <= GRAD_TOL
    assert norm_rel(layer.dw_weight.grad.cpu().numpy().reshape(ci, 3, 3), rddw) <= GRAD_TOL
    if hb:
        assert norm_rel(layer.bias.grad.cpu().numpy(), rdb) <= GRAD_TOL
    if dwb:
        assert norm_rel(layer.dw_bias.grad.cpu().numpy(), rddb) <= GRAD_TOL


TC_DSC = [  # c_in, c_out, cg, co, n, h, w, stride, dw_bias, bias, expect one fused kernel
    (64, 64, 2, "50%", 4, 32, 32, 1, True, True, True),
    (64, 128, 2, "50%", 3, 32, 32, 1, False, True, True),
    (128, 128, 2, "50%", 2, 16, 16, 1, True, False, False),  # two 64-row SCC tiles: the pair
    (128, 128, 2, "25%", 2, 32, 32, 1, True, True, False),  # co = 25 %: several window classes, the pair
    (32, 64, 2, "25%", 3, 16, 16, 1, False, True, True),
    (64, 128, 2, "50%", 2, 16, 16, 1, False, True, True),
    (64, 64, 2, "50%", 2, 16, 32, 1, True, True, True),   # 16 rows of 32
    (64, 64, 2, "50%", 2, 8, 8, 1, False, True, False),   # 8-wide: the depthwise + SCC pair
    (64, 128, 2, "50%", 2, 32, 32, 2, True, True, False),  # stride 2: the pair
]


@pytest.mark.parametrize("case", TC_DSC, ids=lambda c: f"{c[0]}-{c[1]}-cg{c[2]}-{c[3]}-{c[5]}x{c[6]}-s{c[7]}")
def test_dsc_forward_t_matches_oracle(port, case):
    """scc_dsc_forward_t_f32: y = SCC(DW3x3(x)) and t = DW3x3(x) against the
    oracle composition (port.dw_forward -> port.forward, fp64); on stride-1
    16- / 32-wide images one tensor-core kernel (the depthwise stage in its
    staging step) when the SCC layer is one row tile over every channel,
    elsewhere the depthwise kernel + the SCC forward."""
    import paper_2101_00745_b200 as scc
    ci, co, cg, ov, n, h, w, s, dwb, hb, one = case
    cfg = scc.scc_config_new(ci, co, cg, ov, hb)
    x, dww, dwbias = _problem(case[:10], seed=7)
    rng = np.random.default_rng(2)
    gw = cfg.group_width
    wt = rng.uniform(-(1 / gw) ** 0.5, (1 / gw) ** 0.5, co * gw).astype(np.float32)
    b = rng.uniform(-0.5, 0.5, co).astype(np.float32) if hb else None
    wts = scc.SccWeights(torch.from_numpy(wt).cuda(), torch.from_numpy(b).cuda() if hb else None)
    xt, wd = torch.from_numpy(x).cuda(), torch.from_numpy(dww).cuda()
    bd = torch.from_numpy(dwbias).cuda() if dwb else None
    scc.dsc_forward_t(xt, wd, bd, wts, cfg, s)  # plan tables / scratch
    torch.cuda.synchronize()
    before = scc.launch_count()
    y, t = scc.dsc_forward_t(xt, wd, bd, wts, cfg, s)
    torch.cuda.synchronize()
    launched = scc.launch_count() - before
    assert (launched == 1) == one, launched
    rt = port.dw_forward(x, dww, dwbias, 3, s)
    o = port.config(ci, co, cg, ("ratio", float(ov[:-1]) / 100), hb)
    ry = port.forward(o, rt, wt, b)
    assert norm_rel(t.cpu().numpy(), rt) <= FWD_TOL
    assert norm_rel(y.cpu().numpy(), ry) <= FWD_TOL
    y2, t2 = scc.dsc_forward_t(xt, wd, bd, wts, cfg, s)
    assert torch.equal(y, y2) and torch.equal(t, t2)  # deterministic


@pytest.mark.parametrize("case", [TC_DSC[0], TC_DSC[1], TC_DSC[2], TC_DSC[3], TC_DSC[4]], ids=lambda c: f"{c[0]}-{c[1]}-{c[5]}x{c[6]}")
def test_dsc2d_fused_tensor_core_matches_reference(ref, case):
    """DSC2d(fused=True) on the tensor-core fused forward: forward and every
    gradient against the reference's own stages (t from the fused kernel is
    the SCC backward's input)."""
    import paper_2101_00745_b200 as scc
    ci, co, cg, ov, n, h, w, s, dwb, hb, _ = case
    torch.manual_seed(4)
    layer = scc.DSC2d(ci, co, s, cg, ov, dw_bias=dwb, bias=hb, fused=True, device="cuda")
    with torch.no_grad():
        if hb:
            layer.bias.uniform_(-0.5, 0.5)
        if dwb:
            layer.dw_bias.uniform_(-0.5, 0.5)
    x = torch.randn(n, ci, h, w, device="cuda", requires_grad=True)
    y = layer(x)
    gy = torch.randn_like(y)
    y.backward(gy)
    xn = x.detach().cpu().numpy()
    dww = layer.dw_weight.detach().cpu().numpy().reshape(ci, 3, 3)
    dwbn = layer.dw_bias.detach().cpu().numpy() if dwb else None
    wn = layer.weight.detach().cpu().numpy().reshape(-1)
    bn = layer.bias.detach().cpu().numpy() if hb else None
    o = ref.config(ci, co, cg, ov, hb)
    t = ref.dw_forward(xn, dww, dwbn, 3, s)
    ry = ref.forward(o, t, wn, bn)
    gyn = gy.cpu().numpy()
    dt = ref.backward_input(o, gyn, wn)
    rdw, rdb = ref.backward_params(o, gyn, t)
    rdx, rddw, rddb = ref.dw_backward(dt, xn, dww, 3, s, dwb)
    assert norm_rel(y.detach().cpu().numpy(), ry) <= FWD_TOL
    assert norm_rel(x.grad.cpu().numpy(), rdx) <= GRAD_TOL
    assert norm_rel(layer.dw_weight.grad.cpu().numpy().reshape(ci, 3, 3), rddw) <= GRAD_TOL
    assert norm_rel(layer.weight.grad.cpu().numpy().reshape(-1), rdw) <= GRAD_TOL
    if hb:
        assert norm_rel(layer.bias.grad.cpu().numpy(), rdb) <= GRAD_TOL
    if dwb:
        assert norm_rel(layer.dw_bias.grad.cpu().numpy(), rddb) <= GRAD_TOL


def test_dsc_forward_t_ignores_stale_memory():
    """The fused forward's corner taps of a stage's first / last pixel read
    outside the stage; their padding must come from selects, not from a zero
    weight (0 x NaN is NaN).  Shared and global memory left full of NaN by
    earlier work must not reach y or t."""
    import paper_2101_00745_b200 as scc
    cfg = scc.scc_config_new(64, 64, 2, "50%", False)
    wts = scc.scc_weights_init(cfg, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(9)
    x = torch.randn(32, 64, 32, 32, device="cuda", generator=g)
    dw = (torch.rand(64, 1, 3, 3, device="cuda", generator=g) - 0.5) / 3
    y0, t0 = scc.dsc_forward_t(x, dw, None, wts, cfg, 1)
    for _ in range(3):
        junk = torch.full((1 << 26,), float("nan"), device="cuda")
        scc.scc_forward(junk[: x.numel()].view_as(x), wts, cfg)  # NaN through the kernels' shared memory
        del junk
        y, t = scc.dsc_forward_t(x, dw, None, wts, cfg, 1)
        assert torch.isfinite(y).all() and torch.isfinite(t).all()
        assert torch.equal(y, y0) and torch.equal(t, t0)


@pytest.mark.parametrize("shape", [(8, 64, 32, 32, 1), (8, 64, 32, 32, 2), (16, 128, 16, 16, 1), (4, 32, 7, 9, 1)],
                         ids=lambda s: f"{s[1]}ch-{s[2]}x{s[3]}-s{s[4]}")
def test_depthwise_and_dsc_ignore_stale_memory(shape):
    """The depthwise kernels and the CUDA-core fused dsc forward are bitwise
    unchanged after global and shared memory were left full of NaN."""
    import paper_2101_00745_b200 as scc
    n, c, h, w, s = shape
    g = torch.Generator(device="cuda").manual_seed(12)
    x = torch.randn(n, c, h, w, device="cuda", generator=g)
    wt = (torch.rand(c, 1, 3, 3, device="cuda", generator=g) - 0.5) / 3
    b = torch.rand(c, device="cuda", generator=g) - 0.5
    cfg = scc.scc_config_new(c, 2 * c, 2, "50%", True)
    wts = scc.scc_weights_init(cfg, device="cuda")

    def run():
        y = scc.dw3x3_forward(x, wt, b, s)
        gy = torch.ones_like(y) * 0.25 + y
        dx, dw, db = scc.dw3x3_backward(gy, x, wt, s, True)
        dx2 = scc.dw3x3_backward_data(gy, wt, (h, w), s)
        dw2, db2 = scc.dw3x3_backward_weight(gy, x, s, True)
        yd = scc.dsc_forward(x, wt, b, wts, cfg, s)
        yt, t = scc.dsc_forward_t(x, wt, b, wts, cfg, s)
        return [y, dx, dw, db, dx2, dw2, db2, yd, yt, t]

    ref = run()
    for _ in range(2):
        junk = torch.full((1 << 26,), float("nan"), device="cuda")
        v = junk[: x.numel()].view_as(x)
        scc.dw3x3_forward(v, wt, b, s)
        scc.dsc_forward(v, wt, b, wts, cfg, s)
        del junk, v
        for a, r in zip(run(), ref):
            assert torch.equal(a, r)
