"""TEST INFRASTRUCTURE ONLY: ctypes bindings for the two CPU oracles.

See ``oracle/__init__.py``.  Inputs are numpy arrays; they are up-cast to
float64 (exact for float32 data) before the call, as the reference computes in
double (proj/core/include/sccl/tensor.hpp:11-15).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "libscc_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsccl_ref.so")

_i64 = C.c_int64
_i32 = C.c_int32
_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)


class OracleError(RuntimeError):
    """Raised with the reference's status code (1 shape, 2 index, 3 config,
    4 argument, 8 format (fixture files); sccl/errors.hpp:9-55)."""

    def __init__(self, code: int, msg: str = ""):
        super().__init__(f"oracle status {code}: {msg}")
        self.code = code


class _Cfg(C.Structure):
    _fields_ = [
        ("c_in", _i64),
        ("c_out", _i64),
        ("cg", _i64),
        ("overlap_channels", _i64),
        ("group_width", _i64),
        ("shift", _i64),
        ("has_bias", _i32),
    ]


@dataclass(frozen=True)
class OracleConfig:
    c_in: int
    c_out: int
    cg: int
    overlap_channels: int
    group_width: int
    shift: int
    has_bias: bool

    def _c(self) -> _Cfg:
        return _Cfg(self.c_in, self.c_out, self.cg, self.overlap_channels,
                    self.group_width, self.shift, int(self.has_bias))


def build(quiet: bool = True) -> None:
    """Compile the oracles (make -C oracle).  The reference half is skipped
    automatically when /root/reference is absent (prebuilt _ref is used)."""
    out = subprocess.run(["make", "-C", HERE], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


def _d(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


class _Base:
    def _overlap_args(self, overlap):
        """overlap: ('ratio', r) | ('channels', k) | text like '50%'."""
        if isinstance(overlap, str):
            return self.parse_overlap(overlap)
        kind, val = overlap
        if kind == "ratio":
            return 1, float(val), 0
        return 0, 0.0, int(val)

    def forward(self, cfg: OracleConfig, x, w, b):
        x = _d(x)
        n, c, h, wd = x.shape
        y = np.empty((n, cfg.c_out, h, wd), np.float64)
        w = _d(w)
        b = _d(b) if (cfg.has_bias and b is not None) else np.zeros(max(cfg.c_out, 1))
        self._fwd(C.byref(cfg._c()), n, h, wd, _ptr(x), _ptr(w), _ptr(b), _ptr(y))
        return y

    def backward_input(self, cfg: OracleConfig, dy, w):
        dy = _d(dy)
        n, c, h, wd = dy.shape
        dx = np.empty((n, cfg.c_in, h, wd), np.float64)
        w = _d(w)
        self._bwd_in(C.byref(cfg._c()), n, h, wd, _ptr(dy), _ptr(w), _ptr(dx))
        return dx

    def backward_params(self, cfg: OracleConfig, dy, x):
        dy, x = _d(dy), _d(x)
        n, c, h, wd = x.shape
        dw = np.empty(cfg.c_out * cfg.group_width, np.float64)
        db = np.zeros(cfg.c_out, np.float64)
        self._bwd_p(C.byref(cfg._c()), n, h, wd, _ptr(dy), _ptr(x), _ptr(dw), _ptr(db))
        return dw, (db if cfg.has_bias else None)


    def dw_forward(self, x, wt, bias, k=3, stride=1):
        """Depthwise k x k conv of a dsc_block (model.cpp:213-220; padding k/2,
        reference.cpp:74-123).  wt: [c][k][k]; bias: [c] or None."""
        x = _d(x)
        n, c, h, wd = x.shape
        pad = k // 2
        ho, wo = (h + 2 * pad - k) // stride + 1, (wd + 2 * pad - k) // stride + 1
        y = np.empty((n, c, ho, wo), np.float64)
        wt = _d(wt)
        b = _d(bias) if bias is not None else None
        self._dw(n, c, h, wd, k, stride, _ptr(x), _ptr(wt), _ptr(b) if b is not None else None, _ptr(y))
        return y


    def dw_backward(self, dy, x, wt, k=3, stride=1, with_bias=False):
        """grouped_conv_backward of the depthwise stage (groups = c, padding
        k/2; reference.cpp:155-247): (dx, dW [c][k][k], db or None)."""
        if not hasattr(self, "_dwb"):
            raise NotImplementedError("depthwise backward: compiled reference only")
        dy, x, wt = _d(dy), _d(x), _d(wt)
        n, c, h, wd = x.shape
        dx = np.empty_like(x)
        dwt = np.empty(c * k * k, np.float64)
        db = np.empty(c, np.float64) if with_bias else None
        self._dwb(n, c, h, wd, k, stride, _ptr(dy), _ptr(x), _ptr(wt), _ptr(dx), _ptr(dwt),
                  _ptr(db) if db is not None else None)
        return dx, dwt.reshape(c, k, k), db


class PortOracle(_Base):
    """oracle/scc_oracle.c (plain-C restatement, single thread)."""

    kind = "port"

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            build()
        L = self.lib = C.CDLL(path)
        L.scc_oracle_config_new.argtypes = [_i64, _i64, _i64, _i32, C.c_double, _i64,
                                            _i32, C.POINTER(_Cfg)]
        L.scc_oracle_config_new.restype = C.c_int
        L.scc_oracle_overlap_resolve.argtypes = [_i32, C.c_double, _i64, _i64, _i64p]
        L.scc_oracle_cycle.argtypes = [C.POINTER(_Cfg), _i64p]
        L.scc_oracle_cycle.restype = _i64
        L.scc_oracle_covering.argtypes = [C.POINTER(_Cfg), _i64, _i64p]
        L.scc_oracle_covering.restype = _i64
        for name in ("scc_oracle_forward",):
            getattr(L, name).argtypes = [C.POINTER(_Cfg), _i64, _i64, _i64, _dp, _dp, _dp, _dp]
        L.scc_oracle_backward_input.argtypes = [C.POINTER(_Cfg), _i64, _i64, _i64, _dp, _dp, _dp]
        L.scc_oracle_backward_params.argtypes = [C.POINTER(_Cfg), _i64, _i64, _i64, _dp, _dp,
                                                 _dp, _dp]
        L.scc_oracle_forward_macs.argtypes = [C.POINTER(_Cfg), _i64, _i64, _i64]
        L.scc_oracle_forward_macs.restype = C.c_uint64
        self._fwd = L.scc_oracle_forward
        L.scc_oracle_dw_forward.argtypes = [_i64] * 6 + [_dp, _dp, _dp, _dp]
        self._dw = L.scc_oracle_dw_forward
        self._bwd_in = L.scc_oracle_backward_input
        self._bwd_p = L.scc_oracle_backward_params

    def parse_overlap(self, text):  # the port has no text parser; use the reference's
        raise NotImplementedError("Overlap::parse is pinned through RefOracle")

    def config(self, c_in, c_out, cg, overlap, has_bias=True) -> OracleConfig:
        is_ratio, ratio, count = self._overlap_args(overlap)
        c = _Cfg()
        rc = self.lib.scc_oracle_config_new(c_in, c_out, cg, is_ratio, ratio, count,
                                            int(has_bias), C.byref(c))
        if rc:
            raise OracleError(rc, "config")
        return OracleConfig(c.c_in, c.c_out, c.cg, c.overlap_channels, c.group_width,
                            c.shift, bool(c.has_bias))

    def cycle(self, cfg: OracleConfig):
        buf = (C.c_int64 * cfg.c_in)()
        n = self.lib.scc_oracle_cycle(C.byref(cfg._c()), buf)
        return list(buf[:n])

    def covering(self, cfg: OracleConfig, ic: int):
        buf = (C.c_int64 * cfg.c_out)()
        n = self.lib.scc_oracle_covering(C.byref(cfg._c()), ic, buf)
        if n < 0:
            raise OracleError(-n, "covering")
        return list(buf[:n])

    def forward_macs(self, cfg: OracleConfig, n, h, w) -> int:
        return int(self.lib.scc_oracle_forward_macs(C.byref(cfg._c()), n, h, w))


class RefOracle(_Base):
    """The compiled reference (oracle/_ref/libsccl_ref.so via ref_shim.cpp)."""

    kind = "reference"

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_set_num_threads.argtypes = [C.c_int]
        L.ref_num_threads.restype = C.c_int
        L.ref_overlap_parse.argtypes = [C.c_char_p, C.POINTER(_i32), C.POINTER(C.c_double),
                                        _i64p]
        L.ref_overlap_resolve.argtypes = [_i32, C.c_double, _i64, _i64, _i64p]
        L.ref_config_new.argtypes = [_i64, _i64, _i64, _i32, C.c_double, _i64, _i32,
                                     C.POINTER(_Cfg)]
        L.ref_cycle.argtypes = [C.POINTER(_Cfg), _i64p]
        L.ref_cycle.restype = _i64
        L.ref_window_of.argtypes = [C.POINTER(_Cfg), _i64, _i64p]
        L.ref_covering.argtypes = [C.POINTER(_Cfg), _i64, _i64p, _i64p]
        L.ref_forward.argtypes = [C.POINTER(_Cfg), _i64, _i64, _i64, _dp, _dp, _dp, _dp]
        L.ref_forward_nc.argtypes = [C.POINTER(_Cfg), _i64, _i64, _i64, _i64, _dp, _dp, _i64,
                                     _dp, _i64, _dp]
        L.ref_backward_input.argtypes = [C.POINTER(_Cfg), _i64, _i64, _i64, _dp, _dp, _dp]
        L.ref_backward_params.argtypes = [C.POINTER(_Cfg), _i64, _i64, _i64, _dp, _dp, _dp,
                                          _dp]
        L.ref_problem_new.argtypes = [C.POINTER(_Cfg), _i64, _i64, _i64, _dp, _dp, _dp, _dp]
        L.ref_problem_new.restype = C.c_void_p
        L.ref_problem_step.argtypes = [C.c_void_p]
        L.ref_problem_step.restype = C.c_double
        L.ref_problem_free.argtypes = [C.c_void_p]
        self._fwd = self._checked(L.ref_forward)
        L.sccl_ref_dw_forward.argtypes = [_i64] * 6 + [_dp, _dp, _dp, _dp]
        self._dw = self._checked(L.sccl_ref_dw_forward)
        L.sccl_ref_dw_backward.argtypes = [_i64] * 6 + [_dp] * 6
        self._dwb = self._checked(L.sccl_ref_dw_backward)
        L.ref_fixture_write.argtypes = [C.c_char_p, _i64, _i64, _i64, _i64, _dp]
        L.ref_fixture_read.argtypes = [C.c_char_p, _i64p, _dp, _i64]
        L.ref_fixture_probes.argtypes = [C.c_char_p, C.c_uint64]
        L.ref_compose_forward.argtypes = [C.POINTER(_Cfg), _i32, _i32, _i64, _i64, _i64, _dp, _dp,
                                          _dp, _dp, _i64p]
        L.ref_compose_backward.argtypes = [C.POINTER(_Cfg), _i32, _i32, _i64, _i64, _i64, _dp,
                                           _dp, _dp, _dp, _dp, _dp]
        self._bwd_in = self._checked(L.ref_backward_input)
        self._bwd_p = self._checked(L.ref_backward_params)

    def _checked(self, fn):
        def call(*a):
            rc = fn(*a)
            if rc:
                raise OracleError(rc, self.lib.ref_last_error().decode())
        return call

    def set_num_threads(self, t: int) -> None:
        self._checked(self.lib.ref_set_num_threads)(t)

    def num_threads(self) -> int:
        return int(self.lib.ref_num_threads())

    def parse_overlap(self, text: str):
        r, ratio, count = _i32(), C.c_double(), _i64()
        rc = self.lib.ref_overlap_parse(text.encode(), C.byref(r), C.byref(ratio), C.byref(count))
        if rc:
            raise OracleError(rc, self.lib.ref_last_error().decode())
        return int(r.value), float(ratio.value), int(count.value)

    def resolve(self, overlap, group_width: int) -> int:
        is_ratio, ratio, count = self._overlap_args(overlap)
        out = _i64()
        self._checked(self.lib.ref_overlap_resolve)(is_ratio, ratio, count, group_width,
                                                    C.byref(out))
        return int(out.value)

    def config(self, c_in, c_out, cg, overlap, has_bias=True) -> OracleConfig:
        is_ratio, ratio, count = self._overlap_args(overlap)
        c = _Cfg()
        self._checked(self.lib.ref_config_new)(c_in, c_out, cg, is_ratio, ratio, count,
                                               int(has_bias), C.byref(c))
        return OracleConfig(c.c_in, c.c_out, c.cg, c.overlap_channels, c.group_width,
                            c.shift, bool(c.has_bias))

    def cycle(self, cfg: OracleConfig):
        buf = (C.c_int64 * cfg.c_in)()
        n = self.lib.ref_cycle(C.byref(cfg._c()), buf)
        return list(buf[:n])

    def window_of(self, cfg: OracleConfig, oc: int) -> int:
        out = _i64()
        self._checked(self.lib.ref_window_of)(C.byref(cfg._c()), oc, C.byref(out))
        return int(out.value)

    def covering(self, cfg: OracleConfig, ic: int):
        buf = (C.c_int64 * max(cfg.c_out, 1))()
        n = _i64()
        self._checked(self.lib.ref_covering)(C.byref(cfg._c()), ic, buf, C.byref(n))
        return list(buf[: n.value])

    def forward_shape_probe(self, cfg: OracleConfig, x, w, b):
        """scc_forward with arbitrary extents, so shape errors surface."""
        x, w = _d(x), _d(w)
        b = _d(b) if b is not None else np.zeros(0)
        n, c, h, wd = x.shape
        y = np.empty((n, cfg.c_out, h, wd), np.float64)
        self._checked(self.lib.ref_forward_nc)(C.byref(cfg._c()), n, c, h, wd, _ptr(x),
                                               _ptr(w), w.size, _ptr(b) if b.size else
                                               _ptr(np.zeros(1)), b.size, _ptr(y))
        return y

    # --- DSX1 fixtures (fixture.cpp:29-97) ---
    def fixture_write(self, t, path: str) -> None:
        t = _d(t)
        n, c, h, w = t.shape
        self._checked(self.lib.ref_fixture_write)(path.encode(), n, c, h, w, _ptr(t))

    def fixture_read(self, path: str) -> np.ndarray:
        dims = (C.c_int64 * 4)()
        self._checked(self.lib.ref_fixture_read)(path.encode(), dims, None, 0)
        out = np.empty(tuple(dims), np.float64)
        self._checked(self.lib.ref_fixture_read)(path.encode(), dims, _ptr(out), out.size)
        return out

    def fixture_probes(self, directory: str, seed: int) -> None:
        """The reference CLI's golden probes (tools/scc/main.cpp:98-132), plus
        each probe's input / weight / bias."""
        self._checked(self.lib.ref_fixture_probes)(directory.encode(), seed)

    # --- composition routes (reference.cpp:335-490) ---
    def compose_forward(self, cfg: OracleConfig, route: str, use_cc: bool, x, w, b):
        x, w = _d(x), _d(w)
        b = _d(b) if b is not None else np.zeros(max(cfg.c_out, 1))
        n, _, h, wd = x.shape
        y = np.empty((n, cfg.c_out, h, wd), np.float64)
        aux = _i64()
        self._checked(self.lib.ref_compose_forward)(C.byref(cfg._c()), int(route == "conv"),
                                                    int(use_cc), n, h, wd, _ptr(x), _ptr(w),
                                                    _ptr(b), _ptr(y), C.byref(aux))
        return y, int(aux.value)

    def compose_backward(self, cfg: OracleConfig, route: str, use_cc: bool, dy, x, w):
        dy, x, w = _d(dy), _d(x), _d(w)
        n, _, h, wd = x.shape
        dx = np.empty_like(x)
        dw = np.empty(cfg.c_out * cfg.group_width, np.float64)
        db = np.zeros(max(cfg.c_out, 1), np.float64)
        self._checked(self.lib.ref_compose_backward)(C.byref(cfg._c()), int(route == "conv"),
                                                     int(use_cc), n, h, wd, _ptr(dy), _ptr(x),
                                                     _ptr(w), _ptr(dx), _ptr(dw), _ptr(db))
        return dx, dw, (db[: cfg.c_out] if cfg.has_bias else None)

    # --- timed baseline (bench.py --impl reference / cpu_baseline) ---
    def problem(self, cfg: OracleConfig, x, w, b, dy):
        keep = [_d(x), _d(w), _d(b) if b is not None else np.zeros(cfg.c_out), _d(dy)]
        n, c, h, wd = keep[0].shape
        hnd = self.lib.ref_problem_new(C.byref(cfg._c()), n, h, wd, *(map(_ptr, keep)))
        if not hnd:
            raise OracleError(7, self.lib.ref_last_error().decode())
        return _Problem(self.lib, hnd, keep)


class _Problem:
    def __init__(self, lib, hnd, keep):
        self.lib, self.hnd, self._keep = lib, hnd, keep

    def step(self) -> float:
        return float(self.lib.ref_problem_step(self.hnd))

    def __del__(self):
        if getattr(self, "hnd", None):
            self.lib.ref_problem_free(self.hnd)
            self.hnd = None


def load_port() -> PortOracle:
    return PortOracle()


def load_ref():
    """The compiled reference, or None when oracle/_ref was never built."""
    try:
        return RefOracle()
    except (FileNotFoundError, OSError):
        return None
