"""Probe of the tcgen05 building blocks (tests/cuda/tc_probe.cu): TMA
SWIZZLE_128B MN-major A, manually swizzled K-major B, kind::tf32 MMA, TMEM
epilogue.  Establishes how the tensor core reduces raw fp32 operands to tf32
(the 3xTF32 split in the SCC kernels depends on it) and that the split reaches
~1e-6 norm-relative error."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

from conftest import norm_rel

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "cuda", "_build", "tc_probe.so")


@pytest.fixture(scope="module")
def probe():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(SO):
        os.makedirs(os.path.dirname(SO), exist_ok=True)
        subprocess.check_call([
            "nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-std=c++17",
            "-Xcompiler", "-fPIC", "-shared",
            "-I" + os.path.join(os.path.dirname(HERE), "paper_2101_00745_b200", "csrc"),
            "-o", SO, os.path.join(HERE, "cuda", "tc_probe.cu")])
    lib = C.CDLL(SO)
    lib.tc_probe.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
    return lib


def run(probe, x, w, mode):
    xt = torch.from_numpy(x).cuda()
    wt = torch.from_numpy(w).cuda()
    out = torch.empty(128, 128, device="cuda")
    assert probe.tc_probe(xt.data_ptr(), wt.data_ptr(), out.data_ptr(), mode) == 0
    return out.cpu().numpy()


def trunc(a):
    return (a.view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)


def test_tf32_operand_reduction(probe):
    x = np.full((32, 128), 1.0 + 3 * 2.0 ** -12, np.float32)
    w = np.ones((128, 32), np.float32)
    d = run(probe, x, w, 0)
    # truncation -> exactly 32; round-to-nearest would give 32 * (1 + 2^-10)
    print("raw-operand MMA result", d[0, 0])
    assert d[0, 0] == 32.0


def test_layouts_and_3xtf32(probe):
    rng = np.random.default_rng(0)
    x = rng.standard_normal((32, 128)).astype(np.float32)
    w = rng.standard_normal((128, 32)).astype(np.float32)
    want = (x.astype(np.float64).T @ w.astype(np.float64).T)  # [p][oc]
    d0 = run(probe, x, w, 0)
    want_t = trunc(x).astype(np.float64).T @ trunc(w).astype(np.float64).T
    assert norm_rel(d0, want_t) < 1e-5, norm_rel(d0, want_t)  # layout + truncation
    d1 = run(probe, x, w, 1)
    e = norm_rel(d1, want)
    print("3xTF32 norm-relative error", e)
    assert e < 2e-6
