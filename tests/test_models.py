"""Model-path coverage: every SCC layer shape of SCC-ResNet-18 / SCC-VGG16
(PAPER.md:351-365 via SURVEY.md section 7.3) through the kernels against a
torch fp64 dense reference of the same operator (a masked 1x1 conv), the
parameter counts the paper states, and a short training run whose loss
falls (the BASELINE C2/C3 harness, paper_2101_00745_b200/train.py)."""
import pytest

torch = pytest.importorskip("torch")

import paper_2101_00745_b200 as scc  # noqa: E402
from paper_2101_00745_b200 import models  # noqa: E402

FWD_TOL, GRAD_TOL = 1e-5, 1e-4


def test_param_counts_match_paper():
    # SCC-VGG16 0.87 M, SCC-ResNet-18 0.84 M parameters
    r = models.param_counts(models.SCCResNet18())
    v = models.param_counts(models.SCCVGG16())
    assert r["scc"] == 610304 and abs(r["total"] - 0.84e6) / 0.84e6 < 0.02
    assert v["scc"] == 817152 and abs(v["total"] - 0.87e6) / 0.87e6 < 0.02
    assert len(models.scc_layers(models.SCCResNet18())) == 16


def test_resnet50_param_count_matches_paper():
    # SCC-ResNet-50 12.87 M parameters (CIFAR-10 head).  With the
    # ImageNet 7x7 stem the count is 7,680 higher.
    r = models.param_counts(models.SCCResNet50(num_classes=10))
    assert abs(r["total"] - 12.87e6) / 12.87e6 < 0.002, r
    assert len(models.scc_layers(models.SCCResNet50())) == 16
    assert len(models.scc_layers(models.SCCResNet50(rule="all"))) == 48


# (c_in, c_out, plane) of every SCC layer of SCC-ResNet-50 at 224x224, both rules
RESNET50_SHAPES = [(64, 64, 56), (128, 128, 28), (256, 256, 14), (512, 512, 7),
                   (64, 256, 56), (256, 64, 56), (256, 128, 56), (128, 512, 28), (512, 128, 28),
                   (512, 256, 28), (256, 1024, 14), (1024, 256, 14), (1024, 512, 14),
                   (512, 2048, 7), (2048, 512, 7)]


def _shapes():
    out = set(RESNET50_SHAPES)
    for name, cls in models.MODELS.items():
        if name.startswith("resnet50"):
            continue
        m = cls()
        size = {"resnet18": [32, 32, 16, 16, 8, 8, 4, 4], "vgg16": [32, 16, 16, 8, 8, 8, 4, 4, 4, 2, 2, 2]}[name]
        for layer, hw in zip(models.scc_layers(m), [s for s in size for _ in range(2)] if name == "resnet18" else size):
            out.add((layer.cfg.c_in, layer.cfg.c_out, hw))
    return sorted(out)


def _dense(cfg, w):
    ci, co, gw = cfg.c_in, cfg.c_out, cfg.group_width
    idx = torch.tensor([[((oc * cfg.shift) % ci + s) % ci for s in range(gw)] for oc in range(co)],
                       device=w.device)
    full = torch.zeros(co, ci, device=w.device, dtype=torch.float64)
    full.scatter_add_(1, idx, w.view(co, gw).double())
    return full, idx


@pytest.mark.gpu
@pytest.mark.parametrize("shape", _shapes(), ids=lambda s: f"{s[0]}to{s[1]}_{s[2]}x{s[2]}")
def test_model_layer_shapes(shape):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ci, co, hw = shape
    cfg = scc.scc_config_new(ci, co, 2, "50%", True)
    n = 8 if hw <= 32 else 2
    g = torch.Generator(device="cuda").manual_seed(ci * 7 + co + hw)
    x = torch.randn(n, ci, hw, hw, device="cuda", generator=g)
    gy = torch.randn(n, co, hw, hw, device="cuda", generator=g)
    wts = scc.scc_weights_init(cfg)
    wts.bias.uniform_(-0.5, 0.5)
    y = scc.scc_forward(x, wts, cfg)
    gr = scc.scc_backward(gy, x, wts, cfg)
    W, idx = _dense(cfg, wts.weight)
    yr = torch.einsum("oc,nchw->nohw", W, x.double()) + wts.bias.double().view(1, -1, 1, 1)
    dxr = torch.einsum("oc,nohw->nchw", W, gy.double())
    dwr = torch.gather(torch.einsum("nohw,nchw->oc", gy.double(), x.double()), 1, idx).reshape(-1)
    dbr = gy.double().sum((0, 2, 3))

    def nrel(a, b):
        return float((a.double() - b).abs().max() / b.abs().max())

    assert nrel(y, yr) <= FWD_TOL
    assert nrel(gr.grad_input, dxr) <= GRAD_TOL
    assert nrel(gr.params.grad_weight, dwr) <= GRAD_TOL
    assert nrel(gr.params.grad_bias, dbr) <= GRAD_TOL


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["resnet18", "vgg16", "resnet50"])
def test_training_loss_falls(name):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2101_00745_b200.train import train_throughput
    kw = dict(image=64, num_classes=10) if name == "resnet50" else {}
    # ResNet-50 from scratch hovers near its first loss for ~15 steps at batch
    # 32 (measured 2.49-2.61 vs 2.57 across runs: stock cuDNN convolutions are
    # not bitwise reproducible); by 30 steps it is at ~2.15
    steps = 30 if name == "resnet50" else 15
    r = train_throughput(name, batch=32, steps=steps, warmup=1, **kw)
    assert r["images_per_s"] > 0
    assert r["loss_last"] < r["loss_first"], r
