"""Host-side mirror of the reference SCC operator API, over libscc_b200.

Same names, argument meaning and error behaviour as proj/core's C++ API
(``sccl::Overlap`` / ``scc_config_new`` config.hpp:12-61, ``compute_channel_cycle``
/ ``window_of`` / ``covering_filters`` cycle.hpp:38-48, ``scc_forward`` /
``scc_backward_input`` / ``scc_backward_params`` / ``scc_backward`` kernel.hpp:37-72),
but the tensors are fp32 NCHW ``torch`` CUDA tensors and every operator call
goes through the C ABI into the sm_100a kernels.  torch is only the device
memory / stream plumbing; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import List, Optional

import torch

from . import _lib
from ._lib import (  # noqa: F401  (re-exported error types)
    ArgumentError,
    ConfigError,
    CudaError,
    IndexError_ as IndexError,  # noqa: A001 - sccl::IndexError
    NumericError,
    SccError,
    ShapeError,
    check,
    lib,
)


class Overlap:
    """sccl::Overlap (config.hpp:12-38)."""

    def __init__(self, is_ratio: bool, ratio: float = 0.0, count: int = 0):
        self._is_ratio, self._ratio, self._count = bool(is_ratio), float(ratio), int(count)

    @staticmethod
    def ratio(r: float) -> "Overlap":
        return Overlap(True, r, 0)

    @staticmethod
    def channels(count: int) -> "Overlap":
        return Overlap(False, 0.0, count)

    @staticmethod
    def parse(text: str) -> "Overlap":
        """Overlap::parse (config.cpp:15-37); ArgumentError on bad text."""
        kind, ratio, count = C.c_int32(), C.c_double(), C.c_int64()
        check(lib().scc_overlap_parse(text.encode(), C.byref(kind), C.byref(ratio),
                                      C.byref(count)))
        return Overlap(kind.value == _lib.SCC_OVERLAP_RATIO, ratio.value, count.value)

    def is_ratio(self) -> bool:
        return self._is_ratio

    def resolve(self, group_width: int) -> int:
        """Overlap::resolve (config.cpp:39-53); ConfigError when out of range."""
        out = C.c_int64()
        check(lib().scc_overlap_resolve(self._kind(), self._ratio, self._count, group_width,
                                        C.byref(out)))
        return out.value

    def str(self) -> str:
        if not self._is_ratio:
            return str(self._count)
        return f"{self._ratio * 100.0:g}%"

    def _kind(self) -> int:
        return _lib.SCC_OVERLAP_RATIO if self._is_ratio else _lib.SCC_OVERLAP_CHANNELS

    def __repr__(self) -> str:
        return f"Overlap({self.str()})"


class SccConfig:
    """sccl::SccConfig (config.hpp:43-55) backed by a native plan handle."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)
        c = _lib.ScccConfig()
        check(lib().scc_plan_config(self._h, C.byref(c)))
        self.c_in, self.c_out, self.cg = c.c_in, c.c_out, c.cg
        self.overlap_channels, self.group_width, self.shift = (
            c.overlap_channels, c.group_width, c.shift)
        self.has_bias = bool(c.has_bias)
        self.cyclic_dist = c.cyclic_dist
        self._fully = bool(c.fully_overlapped)
        self._ws_cache = {}

    def fully_overlapped(self) -> bool:
        return self._fully

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def set_path(self, path: int) -> None:
        """Force the kernel family (_lib.SCC_PATH_*) for this layer."""
        check(lib().scc_plan_set_path(self._h, int(path)))
        self._ws_cache.clear()  # the workspace size depends on the family

    def path_for(self, n: int, h: int, w: int) -> int:
        out = C.c_int32()
        check(lib().scc_plan_get_path(self._h, n, h, w, C.byref(out)))
        return out.value

    def workspace_bytes(self, n: int, h: int, w: int) -> int:
        key = (n, h, w)
        if key not in self._ws_cache:
            out = C.c_size_t()
            check(lib().scc_backward_weight_workspace_size(self._h, n, h, w, C.byref(out)))
            self._ws_cache[key] = out.value
        return self._ws_cache[key]

    def __del__(self):
        h = getattr(self, "_h", None)
        L = getattr(_lib, "_lib", None) if _lib is not None else None
        if h is not None and h.value and L is not None:
            L.scc_plan_destroy(h)
            self._h = None

    def __repr__(self) -> str:
        return (f"SccConfig(c_in={self.c_in}, c_out={self.c_out}, cg={self.cg}, "
                f"overlap_channels={self.overlap_channels}, group_width={self.group_width}, "
                f"shift={self.shift}, has_bias={self.has_bias})")


def scc_config_new(c_in: int, c_out: int, cg: int, co, has_bias: bool = True) -> SccConfig:
    """scc_config_new (config.cpp:62-83).  ``co`` is an Overlap or its text."""
    if isinstance(co, str):
        co = Overlap.parse(co)
    h = C.c_void_p()
    check(lib().scc_plan_create(int(c_in), int(c_out), int(cg), co._kind(), co._ratio,
                                co._count, int(bool(has_bias)), C.byref(h)))
    return SccConfig(h.value)


@dataclass(frozen=True)
class ChannelWindow:
    """sccl::ChannelWindow (cycle.hpp:13-26)."""

    start: int
    length: int

    def contains(self, ch: int, c_in: int) -> bool:
        return (ch - self.start + c_in) % c_in < self.length

    def last(self, c_in: int) -> int:
        return (self.start + self.length - 1) % c_in


@dataclass(frozen=True)
class ChannelCycle:
    """sccl::ChannelCycle (cycle.hpp:30-33)."""

    windows: List[ChannelWindow]
    cyclic_dist: int


def compute_channel_cycle(cfg: SccConfig) -> ChannelCycle:
    n = C.c_int64()
    buf = (C.c_int64 * max(cfg.c_in, 1))()
    check(lib().scc_plan_cycle_starts(cfg.handle, buf, cfg.c_in, C.byref(n)))
    wins = [ChannelWindow(int(buf[i]), cfg.group_width) for i in range(n.value)]
    return ChannelCycle(wins, n.value)


def window_of(cycle: ChannelCycle, oc: int) -> ChannelWindow:
    """window_of (cycle.cpp:23-26); IndexError for oc < 0."""
    if oc < 0:
        raise IndexError(f"output channel must be >= 0, got {oc}")
    return cycle.windows[oc % cycle.cyclic_dist]


def covering_filters(cfg: SccConfig, cycle: Optional[ChannelCycle], ic: int) -> List[int]:
    """covering_filters (cycle.cpp:28-40), computed by the native plan."""
    n = C.c_int64()
    buf = (C.c_int64 * max(cfg.c_out, 1))()
    check(lib().scc_plan_covering_filters(cfg.handle, ic, buf, cfg.c_out, C.byref(n)))
    return [int(buf[i]) for i in range(n.value)]


def scc_forward_macs(cfg: SccConfig, n: int, h: int, w: int) -> int:
    out = C.c_uint64()
    check(lib().scc_forward_macs(cfg.handle, n, h, w, C.byref(out)))
    return out.value


# ---------------------------------------------------------------------------
# tensors


@dataclass
class SccWeights:
    """sccl::SccWeights (kernel.hpp:18-21): weight [c_out*gw] in [oc][k] order
    (window-relative slots), bias [c_out] or None."""

    weight: torch.Tensor
    bias: Optional[torch.Tensor]


@dataclass
class SccParamGradients:
    grad_weight: torch.Tensor
    grad_bias: Optional[torch.Tensor]


@dataclass
class SccGradients:
    grad_input: torch.Tensor
    params: SccParamGradients


def scc_weights_filled(cfg: SccConfig, weight_value: float, bias_value: float = 0.0,
                       device="cuda") -> SccWeights:
    """scc_weights_filled (kernel.cpp:75-80)."""
    w = torch.full((cfg.c_out * cfg.group_width,), float(weight_value), dtype=torch.float32,
                   device=device)
    b = (torch.full((cfg.c_out,), float(bias_value), dtype=torch.float32, device=device)
         if cfg.has_bias else None)
    return SccWeights(w, b)


def scc_weights_init(cfg: SccConfig, generator: Optional[torch.Generator] = None,
                     device="cuda") -> SccWeights:
    """scc_weights_init (kernel.cpp:82-87): U(+-sqrt(1/gw)), bias zero."""
    bound = math.sqrt(1.0 / cfg.group_width)
    w = (torch.rand(cfg.c_out * cfg.group_width, generator=generator, dtype=torch.float32,
                    device="cpu") * 2.0 - 1.0) * bound
    b = torch.zeros(cfg.c_out, dtype=torch.float32) if cfg.has_bias else None
    return SccWeights(w.to(device), b.to(device) if b is not None else None)


def _stream(t: torch.Tensor) -> int:
    return torch.cuda.current_stream(t.device).cuda_stream


def _dev4(t: torch.Tensor, name: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or t.dim() != 4:
        raise ShapeError(f"{name} must be a 4-D NCHW tensor")
    if not t.is_cuda or t.dtype != torch.float32:
        raise ArgumentError(f"{name} must be a float32 CUDA tensor (got {t.dtype} on {t.device})")
    return t.contiguous()


def _check_param(t: Optional[torch.Tensor], name: str, device: Optional[torch.device]) -> None:
    """Parameters are handed to the kernels as raw device pointers: they must be
    float32 CUDA tensors on the activations' device (else ArgumentError)."""
    if t is None:
        return
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float32:
        raise ArgumentError(f"{name} must be a float32 CUDA tensor (got "
                            f"{getattr(t, 'dtype', type(t))} on {getattr(t, 'device', '?')})")
    if device is not None and t.device != device:
        raise ArgumentError(f"{name} is on {t.device}, the activations on {device}")


def _check_weights(wts: SccWeights, cfg: SccConfig, device: Optional[torch.device] = None) -> None:
    """check_weights (kernel.cpp:14-25), plus the device / dtype contract of the
    raw-pointer C ABI."""
    _check_param(wts.weight, "weight", device)
    _check_param(wts.bias, "bias", device)
    want_w = cfg.c_out * cfg.group_width
    if wts.weight.numel() != want_w:
        raise ShapeError(f"weight array has {wts.weight.numel()} entries, config needs {want_w}")
    want_b = cfg.c_out if cfg.has_bias else 0
    have_b = 0 if wts.bias is None else wts.bias.numel()
    if have_b != want_b:
        raise ShapeError(f"bias array has {have_b} entries, config needs {want_b}")


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


def scc_forward(input: torch.Tensor, wts: SccWeights, cfg: SccConfig) -> torch.Tensor:
    """scc_forward (kernel.hpp:43-49)."""
    x = _dev4(input, "input")
    if x.shape[1] != cfg.c_in:
        raise ShapeError(f"input has {x.shape[1]} channels, config expects {cfg.c_in}")
    _check_weights(wts, cfg, x.device)
    n, _, h, w = x.shape
    y = torch.empty((n, cfg.c_out, h, w), dtype=torch.float32, device=x.device)
    wt = wts.weight.contiguous()
    b = wts.bias.contiguous() if wts.bias is not None else None
    check(lib().scc_forward_f32(cfg.handle, n, h, w, x.data_ptr(), wt.data_ptr(), _ptr(b),
                                y.data_ptr(), _stream(x)))
    return y


def dsc_forward(input: torch.Tensor, dw_weight: torch.Tensor, dw_bias: Optional[torch.Tensor],
                wts: SccWeights, cfg: SccConfig, stride: int = 1) -> torch.Tensor:
    """Fused dsc_block forward (model.cpp:213-220): SCC(DW3x3(input)), the
    depthwise output computed inside the SCC kernel (never written to HBM).
    dw_weight: [c_in, 3, 3] (or [c_in, 1, 3, 3]); dw_bias: [c_in] or None;
    padding 1, stride 1 or 2 (conv_forward_impl, reference.cpp:74-123)."""
    x = _dev4(input, "input")
    if x.shape[1] != cfg.c_in:
        raise ShapeError(f"input has {x.shape[1]} channels, config expects {cfg.c_in}")
    if dw_weight.numel() != cfg.c_in * 9:
        raise ShapeError(f"depthwise weight has {dw_weight.numel()} entries, needs {cfg.c_in * 9}")
    if dw_bias is not None and dw_bias.numel() != cfg.c_in:
        raise ShapeError(f"depthwise bias has {dw_bias.numel()} entries, needs {cfg.c_in}")
    _check_param(dw_weight, "dw_weight", x.device)
    _check_param(dw_bias, "dw_bias", x.device)
    _check_weights(wts, cfg, x.device)
    n, _, h, w = x.shape
    ho, wo = (h - 1) // stride + 1, (w - 1) // stride + 1
    y = torch.empty((n, cfg.c_out, ho, wo), dtype=torch.float32, device=x.device)
    dww = dw_weight.contiguous().float()
    dwb = dw_bias.contiguous().float() if dw_bias is not None else None
    wt = wts.weight.contiguous()
    b = wts.bias.contiguous() if wts.bias is not None else None
    check(lib().scc_dsc_forward_f32(cfg.handle, n, h, w, stride, x.data_ptr(), dww.data_ptr(),
                                    _ptr(dwb), wt.data_ptr(), _ptr(b), y.data_ptr(), _stream(x)))
    return y


def dsc_forward_t(input: torch.Tensor, dw_weight: torch.Tensor, dw_bias: Optional[torch.Tensor],
                  wts: SccWeights, cfg: SccConfig, stride: int = 1):
    """dsc_block forward returning (y, t) with t = DW3x3(input), the SCC
    stage's input the block's backward needs (scc_dsc_forward_t_f32): one
    tensor-core kernel when the geometry allows, else the depthwise kernel
    then scc_forward."""
    x = _dev4(input, "input")
    if x.shape[1] != cfg.c_in:
        raise ShapeError(f"input has {x.shape[1]} channels, config expects {cfg.c_in}")
    if dw_weight.numel() != cfg.c_in * 9:
        raise ShapeError(f"depthwise weight has {dw_weight.numel()} entries, needs {cfg.c_in * 9}")
    if dw_bias is not None and dw_bias.numel() != cfg.c_in:
        raise ShapeError(f"depthwise bias has {dw_bias.numel()} entries, needs {cfg.c_in}")
    _check_param(dw_weight, "dw_weight", x.device)
    _check_param(dw_bias, "dw_bias", x.device)
    _check_weights(wts, cfg, x.device)
    n, _, h, w = x.shape
    ho, wo = (h - 1) // stride + 1, (w - 1) // stride + 1
    y = torch.empty((n, cfg.c_out, ho, wo), dtype=torch.float32, device=x.device)
    t = torch.empty((n, cfg.c_in, ho, wo), dtype=torch.float32, device=x.device)
    dww = dw_weight.contiguous().float()
    dwb = dw_bias.contiguous().float() if dw_bias is not None else None
    wt = wts.weight.contiguous()
    b = wts.bias.contiguous() if wts.bias is not None else None
    check(lib().scc_dsc_forward_t_f32(cfg.handle, n, h, w, stride, x.data_ptr(), dww.data_ptr(),
                                      _ptr(dwb), wt.data_ptr(), _ptr(b), y.data_ptr(), t.data_ptr(),
                                      _stream(x)))
    return y, t


def _dw_out(h: int, w: int, stride: int):
    return (h - 1) // stride + 1, (w - 1) // stride + 1


def dw3x3_forward(x: torch.Tensor, weight: torch.Tensor, bias: Optional[torch.Tensor],
                  stride: int = 1) -> torch.Tensor:
    """Depthwise 3x3 stage of a dsc_block (groups = c, padding 1;
    conv_forward_impl, reference.cpp:74-123) on the B200 kernels."""
    x = _dev4(x, "input")
    n, c, h, w = x.shape
    if weight.numel() != c * 9:
        raise ShapeError(f"depthwise weight has {weight.numel()} entries, needs {c * 9}")
    ho, wo = _dw_out(h, w, stride)
    y = torch.empty((n, c, ho, wo), dtype=torch.float32, device=x.device)
    wt = weight.contiguous()
    b = bias.contiguous() if bias is not None else None
    check(lib().scc_dw3x3_forward_f32(n, c, h, w, stride, x.data_ptr(), wt.data_ptr(), _ptr(b),
                                      y.data_ptr(), _stream(x)))
    return y


def dw3x3_backward_data(grad_out: torch.Tensor, weight: torch.Tensor, in_hw, stride: int = 1) -> torch.Tensor:
    g = _dev4(grad_out, "grad_out")
    n, c, _, _ = g.shape
    h, w = in_hw
    dx = torch.empty((n, c, h, w), dtype=torch.float32, device=g.device)
    wt = weight.contiguous()
    check(lib().scc_dw3x3_backward_data_f32(n, c, h, w, stride, g.data_ptr(), wt.data_ptr(),
                                            dx.data_ptr(), _stream(g)))
    return dx


def dw3x3_backward_weight(grad_out: torch.Tensor, x: torch.Tensor, stride: int = 1,
                          with_bias: bool = False):
    g, x = _dev4(grad_out, "grad_out"), _dev4(x, "input")
    n, c, h, w = x.shape
    dw = torch.empty((c, 3, 3), dtype=torch.float32, device=x.device)
    db = torch.empty(c, dtype=torch.float32, device=x.device) if with_bias else None
    nb = C.c_size_t()
    check(lib().scc_dw3x3_workspace_size(c, C.byref(nb)))
    ws = torch.empty(max(nb.value, 4), dtype=torch.uint8, device=x.device)
    check(lib().scc_dw3x3_backward_weight_f32(n, c, h, w, stride, g.data_ptr(), x.data_ptr(),
                                              dw.data_ptr(), _ptr(db), ws.data_ptr(), ws.numel(),
                                              _stream(x)))
    return dw, db


def dw3x3_backward(grad_out: torch.Tensor, x: torch.Tensor, weight: torch.Tensor, stride: int = 1,
                   with_bias: bool = False):
    """The whole depthwise backward (grouped_conv_backward, reference.cpp:
    155-247): (dx, dweight [c,3,3], dbias or None), one pass over grad_out
    and x at stride 1 (scc_dw3x3_backward_f32)."""
    g, x = _dev4(grad_out, "grad_out"), _dev4(x, "input")
    n, c, h, w = x.shape
    if weight.numel() != c * 9:
        raise ShapeError(f"depthwise weight has {weight.numel()} entries, needs {c * 9}")
    dx = torch.empty_like(x)
    dw = torch.empty((c, 3, 3), dtype=torch.float32, device=x.device)
    db = torch.empty(c, dtype=torch.float32, device=x.device) if with_bias else None
    nb = C.c_size_t()
    check(lib().scc_dw3x3_workspace_size(c, C.byref(nb)))
    ws = torch.empty(max(nb.value, 4), dtype=torch.uint8, device=x.device)
    wt = weight.contiguous()
    check(lib().scc_dw3x3_backward_f32(n, c, h, w, stride, g.data_ptr(), x.data_ptr(), wt.data_ptr(),
                                       dx.data_ptr(), dw.data_ptr(), _ptr(db), ws.data_ptr(), ws.numel(),
                                       _stream(x)))
    return dx, dw, db


def scc_backward_input(grad_out: torch.Tensor, wts: SccWeights, cfg: SccConfig) -> torch.Tensor:
    """scc_backward_input (kernel.hpp:56-61)."""
    g = _dev4(grad_out, "grad_out")
    if g.shape[1] != cfg.c_out:
        raise ShapeError(f"grad_out has {g.shape[1]} channels, config expects {cfg.c_out}")
    _check_weights(wts, cfg, g.device)
    n, _, h, w = g.shape
    dx = torch.empty((n, cfg.c_in, h, w), dtype=torch.float32, device=g.device)
    wt = wts.weight.contiguous()
    check(lib().scc_backward_data_f32(cfg.handle, n, h, w, g.data_ptr(), wt.data_ptr(),
                                      dx.data_ptr(), _stream(g)))
    return dx


def _check_pair(g: torch.Tensor, x: torch.Tensor, cfg: SccConfig) -> None:
    if (g.shape[1] != cfg.c_out or x.shape[1] != cfg.c_in or g.shape[0] != x.shape[0]
            or g.shape[2:] != x.shape[2:]):
        raise ShapeError("grad_out/input shapes inconsistent with config")


def scc_backward_params(grad_out: torch.Tensor, input: torch.Tensor,
                        cfg: SccConfig) -> SccParamGradients:
    """scc_backward_params (kernel.hpp:62-68)."""
    g, x = _dev4(grad_out, "grad_out"), _dev4(input, "input")
    _check_pair(g, x, cfg)
    n, _, h, w = x.shape
    dw = torch.empty(cfg.c_out * cfg.group_width, dtype=torch.float32, device=x.device)
    db = torch.empty(cfg.c_out, dtype=torch.float32, device=x.device) if cfg.has_bias else None
    wsb = cfg.workspace_bytes(n, h, w)
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=x.device)
    check(lib().scc_backward_weight_f32(cfg.handle, n, h, w, g.data_ptr(), x.data_ptr(),
                                        dw.data_ptr(), _ptr(db), ws.data_ptr(), wsb, _stream(x)))
    return SccParamGradients(dw, db)


def scc_backward(grad_out: torch.Tensor, input: torch.Tensor, wts: SccWeights,
                 cfg: SccConfig) -> SccGradients:
    """scc_backward (kernel.hpp:70-72)."""
    g, x = _dev4(grad_out, "grad_out"), _dev4(input, "input")
    _check_pair(g, x, cfg)
    _check_weights(wts, cfg, x.device)
    n, _, h, w = x.shape
    dx = torch.empty_like(x)
    dw = torch.empty(cfg.c_out * cfg.group_width, dtype=torch.float32, device=x.device)
    db = torch.empty(cfg.c_out, dtype=torch.float32, device=x.device) if cfg.has_bias else None
    wsb = cfg.workspace_bytes(n, h, w)
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=x.device)
    wt = wts.weight.contiguous()
    check(lib().scc_backward_f32(cfg.handle, n, h, w, g.data_ptr(), x.data_ptr(), wt.data_ptr(),
                                 dx.data_ptr(), dw.data_ptr(), _ptr(db), ws.data_ptr(), wsb,
                                 _stream(x)))
    return SccGradients(dx, SccParamGradients(dw, db))


def launch_count() -> int:
    """Kernels this process has launched through libscc_b200."""
    return int(lib().scc_launch_count())
