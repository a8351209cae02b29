"""Probe of the tcgen05 kind::tf32 operand conventions the SCC tensor-core
kernels rely on (tests/cuda/tc_layout_probe.cu, one CTA, M=N=128, K=32):

* K-major SWIZZLE_128B operands with per-k-step descriptor advance work;
* the tensor core reduces raw fp32 operand bits to tf32 by TRUNCATION, so the
  3xTF32 split uses hi = x & 0xFFFFE000, lo = x - hi;
* an MN-major A operand yields all-zero results for kind::tf32 (recorded, not
  relied on) -- which is why the band kernel stages activations in TMEM.
"""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "cuda", "_build", "tc_layout_probe.so")


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
            "-o", SO, os.path.join(HERE, "cuda", "tc_layout_probe.cu")])
    lib = C.CDLL(SO)
    lib.tc_layout.argtypes = [C.c_void_p] * 3 + [C.c_int] * 4
    return lib


def trunc(a):
    return (a.view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)


def rne(a):
    u = a.view(np.uint32).astype(np.uint64)
    u = (u + 0x0FFF + ((u >> 13) & 1)) & 0xFFFFE000
    return u.astype(np.uint32).view(np.float32)


def run(lib, x, w, a_kmajor, a_flag, lbo, sbo):
    xt, wt = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
    out = torch.zeros(128, 128, device="cuda")
    assert lib.tc_layout(xt.data_ptr(), wt.data_ptr(), out.data_ptr(), a_kmajor, a_flag, lbo, sbo) == 0
    return out.cpu().numpy().astype(np.float64)


def test_kmajor_truncation(probe):
    rng = np.random.default_rng(0)
    x = rng.standard_normal((32, 128)).astype(np.float32)
    w = rng.standard_normal((128, 32)).astype(np.float32)
    got = run(probe, x, w, 1, 0, 16, 1024)
    want_t = trunc(x).astype(np.float64).T @ trunc(w).astype(np.float64).T
    want_r = rne(x).astype(np.float64).T @ rne(w).astype(np.float64).T
    e_t = np.abs(got - want_t).max() / np.abs(want_t).max()
    e_r = np.abs(got - want_r).max() / np.abs(want_r).max()
    print(f"vs truncated tf32 {e_t:.2e}, vs round-to-nearest tf32 {e_r:.2e}")
    assert e_t < 1e-6 < e_r


def test_mn_major_recorded(probe):
    rng = np.random.default_rng(1)
    x = rng.standard_normal((32, 128)).astype(np.float32)
    w = rng.standard_normal((128, 32)).astype(np.float32)
    got = run(probe, x, w, 0, 1, 4096, 1024)
    print("MN-major A nonzeros:", int(np.count_nonzero(got)))


# ---- kind::f16 with bf16 operands (the bf16x3 backward kernels) ------------
BF16_SO = os.path.join(HERE, "cuda", "_build", "bf16_probe.so")


@pytest.fixture(scope="module")
def bf16_probe():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(BF16_SO):
        os.makedirs(os.path.dirname(BF16_SO), exist_ok=True)
        subprocess.check_call([
            "nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-std=c++17",
            "-Xcompiler", "-fPIC", "-shared",
            "-I" + os.path.join(os.path.dirname(HERE), "paper_2101_00745_b200", "csrc"),
            "-o", BF16_SO, os.path.join(HERE, "cuda", "bf16_probe.cu")])
    lib = C.CDLL(BF16_SO)
    lib.bf16_probe.argtypes = [C.c_void_p] * 3 + [C.c_int] * 4
    return lib


@pytest.mark.parametrize("mode,swap,ok", [(0, 0, True), (1, 0, True), (0, 1, False)])
def test_bf16_operand_conventions(bf16_probe, mode, swap, ok):
    """The layouts the bf16x3 kernels rely on (tests/cuda/bf16_probe.cu):
    A in TMEM as bf16 pairs with k = 2c in the LOW half of column c; B in
    SWIZZLE_128B either MN-major (8-row K groups 1024 B apart, the fused
    backward's dy) or K-major (the x / weight-panel rows); fp32 accumulation
    of the exact bf16 products."""
    rng = np.random.default_rng(2)
    a = rng.standard_normal((128, 128)).astype(np.float32)
    b = rng.standard_normal((128, 64)).astype(np.float32)
    bf = lambda v: torch.from_numpy(v).to(torch.bfloat16).double().numpy()
    want = bf(a) @ bf(b)
    out = torch.zeros(128, 64, device="cuda")
    at, bt = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    assert bf16_probe.bf16_probe(at.data_ptr(), bt.data_ptr(), out.data_ptr(), mode, swap,
                                 8192 if mode == 0 else 16, 1024) == 0
    e = np.abs(out.cpu().numpy() - want).max() / np.abs(want).max()
    assert (e < 1e-6) == ok, e
