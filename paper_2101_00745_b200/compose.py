"""The paper's "Base" SCC implementations, built from stock PyTorch operators
on the GPU: the composition routes of the reference
(proj/core/src/reference.cpp:335-490, reference.hpp:86-114).

  * channel stack: materialise every filter's window of input channels as one
    stacked tensor [N, c_out*gw, H, W] (``index_select``), then a grouped 1x1
    convolution with groups = c_out (``F.conv2d``);
  * conv stack: one gw-channel slice and one 1x1 convolution per filter, then
    a channel concat (c_out convolutions);
  * use_cc (the channel-cyclic optimisation, DSXplore section 3): slice only
    the cyclic_dist distinct windows and share them (channel stack: whole
    cycles block-copied; conv stack: filter oc reads slice oc % cyclic_dist).

Gradients come from autograd through the same graph, which is what the
reference's backward routes compute explicitly (grouped-conv backward, then
a scatter-add through the slicing).  These are the baselines the SCC kernels
are measured against (scripts/compose_bench.py, bench.py ``compositions``);
they are not the product path.  ``aux_channels`` mirrors
CompositionStats::aux_channels_stored.
"""
from __future__ import annotations

from typing import Optional, Tuple

import torch
import torch.nn.functional as F

from .scc import SccConfig, compute_channel_cycle


def _window_index(cfg: SccConfig, count: int, device) -> torch.Tensor:
    # cached on the config (built once, outside any CUDA-graph capture)
    cache = cfg.__dict__.setdefault("_compose_idx", {})
    key = (count, str(device))
    if key not in cache:
        cyc = compute_channel_cycle(cfg)
        gw = cfg.group_width
        starts = torch.tensor([cyc.windows[i % cyc.cyclic_dist].start for i in range(count)], dtype=torch.long)
        idx = (starts[:, None] + torch.arange(gw)[None, :]) % cfg.c_in
        cache[key] = idx.reshape(-1).to(device)
    return cache[key]


def channel_stack_forward(x: torch.Tensor, weight: torch.Tensor, bias: Optional[torch.Tensor],
                          cfg: SccConfig, use_cc: bool = False) -> Tuple[torch.Tensor, int]:
    """scc_channel_stack_forward (reference.cpp:335-344, build_channel_stack
    :266-312) -> (y, aux_channels)."""
    gw, co = cfg.group_width, cfg.c_out
    if not use_cc:
        stacked = x.index_select(1, _window_index(cfg, co, x.device))
        aux = co * gw
    else:
        cd = cfg.cyclic_dist
        block = x.index_select(1, _window_index(cfg, cd, x.device))
        reps = -(-co // cd)
        stacked = block.repeat(1, reps, 1, 1)[:, : co * gw]
        aux = cd * gw
    y = F.conv2d(stacked, weight.view(co, gw, 1, 1), bias, groups=co)
    return y, aux


def conv_stack_forward(x: torch.Tensor, weight: torch.Tensor, bias: Optional[torch.Tensor],
                       cfg: SccConfig, use_cc: bool = False) -> Tuple[torch.Tensor, int]:
    """scc_conv_stack_forward (reference.cpp:428-447, build_window_slices
    :396-412) -> (y, aux_channels)."""
    gw, co = cfg.group_width, cfg.c_out
    count = cfg.cyclic_dist if use_cc else co
    idx = _window_index(cfg, count, x.device).view(count, gw)
    slices = [x.index_select(1, idx[i]) for i in range(count)]
    w = weight.view(co, 1, gw, 1, 1)
    outs = [F.conv2d(slices[oc % count], w[oc], None if bias is None else bias[oc:oc + 1]) for oc in range(co)]
    return torch.cat(outs, 1), count * gw


ROUTES = {"channel": channel_stack_forward, "conv": conv_stack_forward}


def compose_backward(route: str, use_cc: bool, dy: torch.Tensor, x: torch.Tensor, weight: torch.Tensor,
                     bias: Optional[torch.Tensor], cfg: SccConfig):
    """scc_channel_stack_backward / scc_conv_stack_backward
    (reference.cpp:346-377, :449-488) -> (dx, dW, db or None)."""
    xr = x.detach().requires_grad_(True)
    wr = weight.detach().requires_grad_(True)
    br = None if bias is None else bias.detach().requires_grad_(True)
    y, _ = ROUTES[route](xr, wr, br, cfg, use_cc)
    ins = [xr, wr] + ([br] if br is not None else [])
    g = torch.autograd.grad(y, ins, grad_outputs=dy)
    return g[0], g[1], (g[2] if br is not None else None)
