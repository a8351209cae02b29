"""The drop-in C++ layer (include/sccl_b200.hpp): the reference's own KATs
written against reference-style names, compiled with g++ and linked to
libscc_b200.so.  CPU: it compiles and fails loudly without a GPU.  GPU: it
passes."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_sccl_shim.cpp")
LIBDIR = os.path.join(ROOT, "paper_2101_00745_b200", "_lib")
EXE = os.path.join(ROOT, "tests", "cpp", "_build", "test_sccl_shim")


def _build():
    os.makedirs(os.path.dirname(EXE), exist_ok=True)
    subprocess.check_call(["g++", "-std=c++20", "-O1", "-I" + os.path.join(ROOT, "include"), SRC,
                           "-o", EXE, "-L" + LIBDIR, "-lscc_b200", "-Wl,-rpath," + LIBDIR])


def test_shim_compiles_and_fails_loudly_without_gpu():
    _build()
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present: see the gpu test")
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=60)
    assert r.returncode != 0
    assert "CudaError" in (r.stderr + r.stdout) or "cuda" in (r.stderr + r.stdout).lower()


@pytest.mark.gpu
def test_shim_reference_kats_on_gpu():
    _build()
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=120)
    print(r.stdout, r.stderr)
    assert r.returncode == 0 and "PASSED" in r.stdout
