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


class _DSCFunction(torch.autograd.Function):
    """dsc_block (model.cpp:213-220): y = SCC(DW3x3(x)), every stage on the
    B200 kernels.

    fused=True : forward is scc_dsc_forward_t_f32: one tensor-core kernel
                 computes t = DW(x) in its staging step, feeds the SCC GEMM
                 and stores t for the backward (stride 1, 16- / 32-wide
                 images, one SCC row tile); other geometries run the
                 depthwise kernel then the SCC forward -- never slower than
                 fused=False.
    fused=False: forward is the depthwise kernel then the SCC tensor-core
                 forward, t kept for backward (the reference's
                 Network::backward also keeps stage inputs, model.cpp:306-380).
    Backward: SCC backward kernels on (dy, t), then the depthwise
    backward-data / backward-weight kernels."""

    @staticmethod
    def forward(ctx, x, dw_weight, dw_bias, weight, bias, cfg, stride, fused):
        wts = _scc.SccWeights(weight.reshape(-1), bias)
        if fused:
            y, t = _scc.dsc_forward_t(x, dw_weight, dw_bias, wts, cfg, stride)
        else:
            t = _scc.dw3x3_forward(x, dw_weight, dw_bias, stride)
            y = _scc.scc_forward(t, wts, cfg)
        ctx.cfg, ctx.stride = cfg, stride
        ctx.has_dwb, ctx.has_bias = dw_bias is not None, bias is not None
        e = torch.empty(0, device=x.device)
        ctx.save_for_backward(x, dw_weight, dw_bias if dw_bias is not None else e, weight,
                              bias if bias is not None else e, t if t is not None else e)
        ctx.saved_t = t is not None
        return y

    @staticmethod
    def backward(ctx, gy):
        x, dw_weight, dw_bias, weight, bias, t = ctx.saved_tensors
        cfg, s = ctx.cfg, ctx.stride
        if not ctx.saved_t:
            t = _scc.dw3x3_forward(x, dw_weight, dw_bias if ctx.has_dwb else None, s)
        wts = _scc.SccWeights(weight.reshape(-1), bias if ctx.has_bias else None)
        g = _scc.scc_backward(gy.contiguous(), t, wts, cfg)
        dt = g.grad_input
        dx = ddw = ddb = None
        need_w = ctx.needs_input_grad[1] or (ctx.has_dwb and ctx.needs_input_grad[2])
        if ctx.needs_input_grad[0] and need_w:
            # one pass over dt and x (stride 1)
            dx, ddw, ddb = _scc.dw3x3_backward(dt, x, dw_weight, s, ctx.has_dwb)
            ddw = ddw.view_as(dw_weight)
        elif ctx.needs_input_grad[0]:
            dx = _scc.dw3x3_backward_data(dt, dw_weight, x.shape[2:], s)
        elif need_w:
            ddw, ddb = _scc.dw3x3_backward_weight(dt, x, s, ctx.has_dwb)
            ddw = ddw.view_as(dw_weight)
        dw = g.params.grad_weight.view_as(weight)
        db = g.params.grad_bias if ctx.has_bias else None
        return dx, ddw, ddb, dw, db, None, None, None


def dsc2d(x, dw_weight, dw_bias, weight, bias, cfg, stride: int = 1, fused: bool = False) -> torch.Tensor:
    return _DSCFunction.apply(x, dw_weight, dw_bias, weight, bias, cfg, stride, fused)


class DSC2d(torch.nn.Module):
    """Fused depthwise-3x3 + SCC block (the reference's "dsc_block",
    model.cpp:213-220: DW stage with groups = c_in, padding 1, no activation,
    then the SCC stage).  Parameters: ``dw_weight`` [c_in, 1, 3, 3] (the
    nn.Conv2d depthwise layout), optional ``dw_bias``, and the SCC layer's
    window-relative ``weight`` [c_out, gw] / ``bias``."""

    def __init__(self, in_channels: int, out_channels: int, stride: int = 1, cg: int = 2,
                 co="50%", dw_bias: bool = False, bias: bool = True, fused: bool = False,
                 device=None):
        super().__init__()
        self.fused = fused
        if stride not in (1, 2):
            raise ValueError("DSC2d supports stride 1 or 2")
        self.stride = stride
        self.cfg = _scc.scc_config_new(in_channels, out_channels, cg, co, bias)
        self.dw_weight = torch.nn.Parameter(torch.empty(in_channels, 1, 3, 3, device=device))
        self.dw_bias = torch.nn.Parameter(torch.zeros(in_channels, device=device)) if dw_bias else None
        self.weight = torch.nn.Parameter(torch.empty(out_channels, self.cfg.group_width, device=device))
        self.bias = torch.nn.Parameter(torch.zeros(out_channels, device=device)) if bias else None
        with torch.no_grad():
            # conv_weights_init fan-in bound for the depthwise stage (cig*k*k = 9),
            # scc_weights_init (kernel.cpp:82-87) for the SCC stage
            self.dw_weight.uniform_(-1.0 / 3.0, 1.0 / 3.0)
            b = math.sqrt(1.0 / self.cfg.group_width)
            self.weight.uniform_(-b, b)

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        return dsc2d(x, self.dw_weight, self.dw_bias, self.weight, self.bias, self.cfg, self.stride,
                     self.fused)
