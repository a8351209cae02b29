"""SCC model zoo (CIFAR-shape SCC-ResNet-18 and SCC-VGG16, ImageNet-shape
SCC-ResNet-50).

The reference's model harness is a sequential JSON-described network of
conv / SCC stages (model.cpp:190-232, the "dsc_block" of model.cpp:213-220:
depthwise 3x3 then SCC, nothing in between).  It has no BN, residuals or
pooling, so it cannot express the paper's VGG / ResNet models; these are
built here from the rule SURVEY.md section 7.3 derives from the paper's
parameter counts:

    every 3x3 conv except the stem -> DW3x3(stride s) + SCC(cg=2, co=50%),
    1x1 shortcut convs stay dense, BN + ReLU after the SCC.

SCC-ResNet-50 (BASELINE config C4): the same rule applied to the bottleneck
(its 3x3 conv becomes DW3x3(stride) + SCC, the 1x1 convs, stem, projection
shortcuts and head stay dense) gives 12,866,314 parameters with a 10-class
head -- the paper's 12.87 M -- so that is the default
(rule="paper").  rule="all" additionally turns every bottleneck 1x1 conv into
an SCC layer (BASELINE's "DW + SCC replacing 1x1 convs" read literally;
8.19 M).  The stage-4 SCC layers run on 7x7 planes (P = 49).

The DW3x3 + SCC pairs run the libscc_b200 kernels (``DSC2d``: depthwise
kernels of scc_dw.cu, SCC tensor-core kernels); BN, pooling, the stem, 1x1
shortcuts and the head are stock PyTorch (library ops off the hot path).
The DW -> SCC pair keeps the reference's ordering (no BN between them), which
is what a fused DW+SCC kernel needs.
"""
from __future__ import annotations

from typing import List

import torch
from torch import nn

from .module import DSC2d, SCC2d


class DSC(DSC2d):
    """dsc_block (model.cpp:213-220): depthwise 3x3 (stride s) then SCC, both
    stages on the libscc_b200 kernels (module.DSC2d; no bias on either stage,
    BN follows).  fused=True: on stride-1 16- / 32-wide layers with one SCC
    row tile the depthwise stage runs inside the SCC tensor-core forward
    (scc_dsc_forward_t_f32), elsewhere the same pair of kernels as
    fused=False."""

    def __init__(self, cin: int, cout: int, stride: int = 1, cg: int = 2, co="50%", device=None):
        super().__init__(cin, cout, stride, cg, co, dw_bias=False, bias=False, fused=True, device=device)


class BasicBlock(nn.Module):
    def __init__(self, cin: int, cout: int, stride: int, cg: int, co, device=None):
        super().__init__()
        self.c1 = DSC(cin, cout, stride, cg, co, device)
        self.b1 = nn.BatchNorm2d(cout, device=device)
        self.c2 = DSC(cout, cout, 1, cg, co, device)
        self.b2 = nn.BatchNorm2d(cout, device=device)
        self.short = None
        if stride != 1 or cin != cout:
            self.short = nn.Sequential(
                nn.Conv2d(cin, cout, 1, stride=stride, bias=False, device=device),
                nn.BatchNorm2d(cout, device=device))

    def forward(self, x):
        y = torch.relu(self.b1(self.c1(x)))
        y = self.b2(self.c2(y))
        return torch.relu(y + (x if self.short is None else self.short(x)))


class SCCResNet18(nn.Module):
    """CIFAR ResNet-18 with every 3x3 conv but the stem as DW3x3 + SCC."""

    def __init__(self, num_classes: int = 10, cg: int = 2, co="50%", device=None):
        super().__init__()
        self.stem = nn.Sequential(nn.Conv2d(3, 64, 3, padding=1, bias=False, device=device),
                                  nn.BatchNorm2d(64, device=device), nn.ReLU())
        blocks: List[nn.Module] = []
        cin = 64
        for cout, stride in ((64, 1), (128, 2), (256, 2), (512, 2)):
            blocks += [BasicBlock(cin, cout, stride, cg, co, device), BasicBlock(cout, cout, 1, cg, co, device)]
            cin = cout
        self.blocks = nn.Sequential(*blocks)
        self.fc = nn.Linear(512, num_classes, device=device)

    def forward(self, x):
        y = self.blocks(self.stem(x))
        return self.fc(torch.flatten(nn.functional.adaptive_avg_pool2d(y, 1), 1))


class SCCVGG16(nn.Module):
    """CIFAR VGG16 (13 conv layers, BN) with every 3x3 conv but the first as
    DW3x3 + SCC."""

    CFG = (64, 64, "M", 128, 128, "M", 256, 256, 256, "M", 512, 512, 512, "M", 512, 512, 512, "M")

    def __init__(self, num_classes: int = 10, cg: int = 2, co="50%", device=None):
        super().__init__()
        layers: List[nn.Module] = []
        cin = 3
        for i, v in enumerate(self.CFG):
            if v == "M":
                layers.append(nn.MaxPool2d(2))
                continue
            conv = (nn.Conv2d(cin, v, 3, padding=1, bias=False, device=device) if i == 0
                    else DSC(cin, v, 1, cg, co, device))
            layers += [conv, nn.BatchNorm2d(v, device=device), nn.ReLU()]
            cin = v
        self.features = nn.Sequential(*layers)
        self.fc = nn.Linear(512, num_classes, device=device)

    def forward(self, x):
        return self.fc(torch.flatten(self.features(x), 1))


class Bottleneck(nn.Module):
    """ResNet-50 bottleneck with SCC in place of both 1x1 convs and DW3x3 + SCC
    in place of the 3x3 conv (stride on the depthwise stage)."""

    expansion = 4

    def __init__(self, cin: int, width: int, stride: int, cg: int, co, device=None, rule: str = "paper"):
        super().__init__()
        cout = width * self.expansion

        def pw(a, b):
            if rule == "all":
                return SCC2d(a, b, cg, co, bias=False, device=device)
            return nn.Conv2d(a, b, 1, bias=False, device=device)

        self.c1 = pw(cin, width)
        self.b1 = nn.BatchNorm2d(width, device=device)
        self.c2 = DSC(width, width, stride, cg, co, device)
        self.b2 = nn.BatchNorm2d(width, device=device)
        self.c3 = pw(width, cout)
        self.b3 = nn.BatchNorm2d(cout, device=device)
        self.short = None
        if stride != 1 or cin != cout:
            self.short = nn.Sequential(
                nn.Conv2d(cin, cout, 1, stride=stride, bias=False, device=device),
                nn.BatchNorm2d(cout, device=device))

    def forward(self, x):
        y = torch.relu(self.b1(self.c1(x)))
        y = torch.relu(self.b2(self.c2(y)))
        y = self.b3(self.c3(y))
        return torch.relu(y + (x if self.short is None else self.short(x)))


class SCCResNet50(nn.Module):
    """ImageNet ResNet-50 (stages 3/4/6/3, widths 64..512, 224x224 input) with
    SCC bottlenecks."""

    def __init__(self, num_classes: int = 1000, cg: int = 2, co="50%", device=None, rule: str = "paper"):
        super().__init__()
        if rule not in ("paper", "all"):
            raise ValueError(f"unknown SCC-ResNet-50 rule {rule!r}")
        self.stem = nn.Sequential(nn.Conv2d(3, 64, 7, stride=2, padding=3, bias=False, device=device),
                                  nn.BatchNorm2d(64, device=device), nn.ReLU(),
                                  nn.MaxPool2d(3, stride=2, padding=1))
        blocks: List[nn.Module] = []
        cin = 64
        for width, n, stride in ((64, 3, 1), (128, 4, 2), (256, 6, 2), (512, 3, 2)):
            for i in range(n):
                blocks.append(Bottleneck(cin, width, stride if i == 0 else 1, cg, co, device, rule))
                cin = width * Bottleneck.expansion
        self.blocks = nn.Sequential(*blocks)
        self.fc = nn.Linear(cin, num_classes, device=device)

    def forward(self, x):
        y = self.blocks(self.stem(x))
        return self.fc(torch.flatten(nn.functional.adaptive_avg_pool2d(y, 1), 1))


def _resnet50_all(num_classes: int = 1000, cg: int = 2, co="50%", device=None):
    return SCCResNet50(num_classes, cg, co, device, rule="all")


MODELS = {"resnet18": SCCResNet18, "vgg16": SCCVGG16, "resnet50": SCCResNet50, "resnet50_all": _resnet50_all}


def scc_layers(model: nn.Module):
    """Every SCC stage (standalone SCC2d or the SCC half of a DSC2d block)."""
    return [m for m in model.modules() if isinstance(m, (SCC2d, DSC2d))]


def param_counts(model: nn.Module):
    scc = sum(m.weight.numel() + (m.bias.numel() if m.bias is not None else 0) for m in scc_layers(model))
    total = sum(p.numel() for p in model.parameters())
    return {"total": total, "scc": scc}
