"""ctypes binding of libscc_b200.so (include/scc_b200.h).

The shared library is built in-tree by ``paper_2101_00745_b200/csrc/Makefile``
(``__graft_entry__.build()``).  There is no fallback: if the library is
missing, importing the operator raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SCC_LIB_PATH") or os.path.join(PKG_DIR, "_lib", "libscc_b200.so")
CSRC = os.path.join(PKG_DIR, "csrc")

SCC_OK = 0
SCC_ERR_SHAPE = 1
SCC_ERR_INDEX = 2
SCC_ERR_CONFIG = 3
SCC_ERR_ARGUMENT = 4
SCC_ERR_NUMERIC = 5
SCC_ERR_CUDA = 6
SCC_ERR_INTERNAL = 7

SCC_OVERLAP_CHANNELS = 0
SCC_OVERLAP_RATIO = 1

SCC_PATH_AUTO = 0
SCC_PATH_CUDA_CORE = 1
SCC_PATH_TENSOR = 2
SCC_PATH_TENSOR_STREAMED = 3

# Every symbol include/scc_b200.h declares (tests assert the .so exports them).
EXPORTS = (
    "scc_last_error", "scc_abi_version", "scc_launch_count", "scc_debug_trace", "scc_debug_trace_fused",
    "scc_overlap_parse", "scc_overlap_resolve",
    "scc_plan_create", "scc_plan_destroy", "scc_plan_config", "scc_plan_cycle_starts",
    "scc_plan_window_of", "scc_plan_covering_filters", "scc_forward_macs",
    "scc_plan_set_path", "scc_plan_get_path",
    "scc_forward_f32", "scc_backward_data_f32", "scc_backward_weight_workspace_size",
    "scc_backward_weight_f32", "scc_backward_f32", "scc_dsc_forward_f32", "scc_dsc_forward_t_f32",
    "scc_dw3x3_forward_f32", "scc_dw3x3_backward_data_f32", "scc_dw3x3_workspace_size",
    "scc_dw3x3_backward_weight_f32", "scc_dw3x3_backward_f32",
    "scc_forward_host_f32", "scc_backward_host_f32", "scc_fwd_bwd_host_f32",
    "scc_backward_data_host_f32", "scc_backward_weight_host_f32",
)


class SccError(RuntimeError):
    """Base error; subclasses mirror sccl/errors.hpp:9-55."""

    code = SCC_ERR_INTERNAL


class ShapeError(SccError):
    code = SCC_ERR_SHAPE


class IndexError_(SccError):  # noqa: N801 - mirrors sccl::IndexError
    code = SCC_ERR_INDEX


class ConfigError(SccError):
    code = SCC_ERR_CONFIG


class ArgumentError(SccError):
    code = SCC_ERR_ARGUMENT


class NumericError(SccError):
    code = SCC_ERR_NUMERIC


class CudaError(SccError):
    code = SCC_ERR_CUDA


_ERRORS = {c.code: c for c in (ShapeError, IndexError_, ConfigError, ArgumentError,
                               NumericError, CudaError)}


class ScccConfig(C.Structure):
    _fields_ = [
        ("c_in", C.c_int64),
        ("c_out", C.c_int64),
        ("cg", C.c_int64),
        ("overlap_channels", C.c_int64),
        ("group_width", C.c_int64),
        ("shift", C.c_int64),
        ("has_bias", C.c_int32),
        ("fully_overlapped", C.c_int32),
        ("cyclic_dist", C.c_int64),
    ]


_lock = threading.Lock()
_lib = None


def build_library(quiet: bool = True) -> str:
    out = subprocess.run(["make", "-C", CSRC, "-j4"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("libscc_b200 build failed:\n" + out.stdout[-4000:] + out.stderr[-4000:])
    if not quiet:
        print(out.stdout)
    return LIB_PATH


def _declare(L):
    i64, i32, vp, fp = C.c_int64, C.c_int32, C.c_void_p, C.c_void_p
    P = C.POINTER
    sig = {
        "scc_last_error": ([], C.c_char_p),
        "scc_abi_version": ([], C.c_int),
        "scc_launch_count": ([], C.c_uint64),
        "scc_debug_trace": ([C.POINTER(C.c_uint64), C.c_int], C.c_int),
        "scc_debug_trace_fused": ([C.POINTER(C.c_uint64), C.c_int], C.c_int),
        "scc_overlap_parse": ([C.c_char_p, P(i32), P(C.c_double), P(i64)], C.c_int),
        "scc_overlap_resolve": ([i32, C.c_double, i64, i64, P(i64)], C.c_int),
        "scc_plan_create": ([i64, i64, i64, i32, C.c_double, i64, i32, P(vp)], C.c_int),
        "scc_plan_destroy": ([vp], C.c_int),
        "scc_plan_config": ([vp, P(ScccConfig)], C.c_int),
        "scc_plan_cycle_starts": ([vp, P(i64), i64, P(i64)], C.c_int),
        "scc_plan_window_of": ([vp, i64, P(i64), P(i64)], C.c_int),
        "scc_plan_covering_filters": ([vp, i64, P(i64), i64, P(i64)], C.c_int),
        "scc_forward_macs": ([vp, i64, i64, i64, P(C.c_uint64)], C.c_int),
        "scc_plan_set_path": ([vp, i32], C.c_int),
        "scc_plan_get_path": ([vp, i64, i64, i64, P(i32)], C.c_int),
        "scc_forward_f32": ([vp, i64, i64, i64, fp, fp, fp, fp, vp], C.c_int),
        "scc_backward_data_f32": ([vp, i64, i64, i64, fp, fp, fp, vp], C.c_int),
        "scc_backward_weight_workspace_size": ([vp, i64, i64, i64, P(C.c_size_t)], C.c_int),
        "scc_backward_weight_f32": ([vp, i64, i64, i64, fp, fp, fp, fp, vp, C.c_size_t, vp],
                                    C.c_int),
        "scc_dsc_forward_f32": ([vp, i64, i64, i64, i64, fp, fp, fp, fp, fp, fp, vp], C.c_int),
        "scc_dsc_forward_t_f32": ([vp, i64, i64, i64, i64, fp, fp, fp, fp, fp, fp, fp, vp], C.c_int),
        "scc_dw3x3_forward_f32": ([i64, i64, i64, i64, i64, fp, fp, fp, fp, vp], C.c_int),
        "scc_dw3x3_backward_data_f32": ([i64, i64, i64, i64, i64, fp, fp, fp, vp], C.c_int),
        "scc_dw3x3_workspace_size": ([i64, P(C.c_size_t)], C.c_int),
        "scc_dw3x3_backward_weight_f32": ([i64, i64, i64, i64, i64, fp, fp, fp, fp, vp, C.c_size_t,
                                           vp], C.c_int),
        "scc_dw3x3_backward_f32": ([i64, i64, i64, i64, i64, fp, fp, fp, fp, fp, fp, vp, C.c_size_t,
                                    vp], C.c_int),
        "scc_backward_f32": ([vp, i64, i64, i64, fp, fp, fp, fp, fp, fp, vp, C.c_size_t, vp],
                             C.c_int),
        "scc_forward_host_f32": ([vp, i64, i64, i64, fp, fp, fp, fp], C.c_int),
        "scc_backward_host_f32": ([vp, i64, i64, i64, fp, fp, fp, fp, fp, fp], C.c_int),
        "scc_fwd_bwd_host_f32": ([vp, i64, i64, i64, fp, fp, fp, fp, fp, fp, fp, fp], C.c_int),
        "scc_backward_data_host_f32": ([vp, i64, i64, i64, fp, fp, fp], C.c_int),
        "scc_backward_weight_host_f32": ([vp, i64, i64, i64, fp, fp, fp, fp], C.c_int),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res


def lib():
    """Load (never silently rebuild on a GPU box) the native library."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise ImportError(
                        f"{LIB_PATH} is missing: run __graft_entry__.build() "
                        "(make -C paper_2101_00745_b200/csrc). There is no CPU fallback.")
                L = C.CDLL(LIB_PATH)
                _declare(L)
                _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != SCC_OK:
        msg = lib().scc_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, SccError)(msg)
