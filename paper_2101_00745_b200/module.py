"""torch.autograd integration of the SCC operator (the model-zoo consumer).

``SCC2d`` plays the role of the reference's SCC network stage
(model.cpp:176, forward call model.cpp:266, backward call model.cpp:372): its
forward and backward run the libscc_b200 kernels, its parameters are the
reference's window-relative weight [c_out][gw] and bias [c_out].
"""
from __future__ import annotations

import math

import torch

from . import scc as _scc


class _SCCFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, weight, bias, cfg):
        wts = _scc.SccWeights(weight.reshape(-1), bias)
        y = _scc.scc_forward(x, wts, cfg)
        ctx.cfg = cfg
        ctx.save_for_backward(x, weight, bias if bias is not None else torch.empty(0))
        ctx.has_bias = bias is not None
        return y

    @staticmethod
    def backward(ctx, gy):
        x, weight, bias = ctx.saved_tensors
        cfg = ctx.cfg
        need_x, need_w, need_b = ctx.needs_input_grad[:3]
        gy = gy.contiguous()
        wts = _scc.SccWeights(weight.reshape(-1), bias if ctx.has_bias else None)
        dx = dw = db = None
        if need_x and (need_w or need_b):
            g = _scc.scc_backward(gy, x, wts, cfg)
            dx, dw, db = g.grad_input, g.params.grad_weight, g.params.grad_bias
        elif need_x:
            dx = _scc.scc_backward_input(gy, wts, cfg)
        elif need_w or need_b:
            p = _scc.scc_backward_params(gy, x, cfg)
            dw, db = p.grad_weight, p.grad_bias
        if dw is not None:
            dw = dw.view_as(weight)
        return dx, dw, (db if ctx.has_bias else None), None


def scc2d(x: torch.Tensor, weight: torch.Tensor, bias, cfg: "_scc.SccConfig") -> torch.Tensor:
    return _SCCFunction.apply(x, weight, bias, cfg)


class SCC2d(torch.nn.Module):
    """Sliding-channel convolution layer: 1x1, stride 1, no padding
    (SPEC.md:257), cg channel groups, overlap co (text like "50%" or a count)."""

    def __init__(self, in_channels: int, out_channels: int, cg: int, co="50%",
                 bias: bool = True, device=None):
        super().__init__()
        self.cfg = _scc.scc_config_new(in_channels, out_channels, cg, co, bias)
        gw = self.cfg.group_width
        self.weight = torch.nn.Parameter(torch.empty(out_channels, gw, device=device))
        self.bias = torch.nn.Parameter(torch.empty(out_channels, device=device)) if bias else None
        self.reset_parameters()

    def reset_parameters(self) -> None:
        # scc_weights_init (kernel.cpp:82-87)
        bound = math.sqrt(1.0 / self.cfg.group_width)
        with torch.no_grad():
            self.weight.uniform_(-bound, bound)
            if self.bias is not None:
                self.bias.zero_()

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        return scc2d(x, self.weight, self.bias, self.cfg)

    def extra_repr(self) -> str:
        c = self.cfg
        return (f"{c.c_in}, {c.c_out}, cg={c.cg}, overlap={c.overlap_channels}, "
                f"group_width={c.group_width}, bias={c.has_bias}")
