"""Reference-harness drop-in: the reference's own network,
dataset and SGD code (proj/core/src/model.cpp, dataset.cpp, train.cpp) linked
against tests/refharness/kernel_b200.cpp -- the sccl::scc_* functions of
kernel.hpp:37-72 implemented over the C ABI -- instead of kernel.cpp.

train_ref (reference kernel.cpp, fp64) and train_b200 (every SCC layer on the
B200 in fp32) run the same seeded work; the whole-network logits and every
stage's gradients agree within the north_star bars (norm-relative: forward
1e-5 per SCC layer, gradients 1e-4; after several fp32 SCC layers the bound is
applied to the network outputs as 1e-4), and SGD training histories agree.
Both binaries are built by __graft_entry__.build() from the reference sources
in place (tests/refharness/Makefile)."""
import json
import os
import subprocess

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
BUILD = os.path.join(HERE, "refharness", "_build")
REF_EXE = os.path.join(BUILD, "train_ref")
GPU_EXE = os.path.join(BUILD, "train_b200")
MODELS = os.path.join(BUILD, "models")  # proj/models/*.json, staged by the Makefile


def _model(name):
    return os.path.join(MODELS, name)


def _need(exe):
    if not os.path.exists(exe):
        pytest.skip(f"{os.path.basename(exe)} not built (needs /root/reference at build time)")


def _nrel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def _grad(exe, model, batch, spatial):
    out = subprocess.run([exe, _model(model), "grad", str(batch), str(spatial)], capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    return json.loads(out.stdout)


def _train(exe, *args):
    out = subprocess.run([exe, *map(str, args)], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    return [tuple(float(t) for t in line.split()[1::2]) for line in out.stdout.splitlines()]


def test_reference_harness_runs_on_cpu():
    """The reference build of the harness itself (no GPU): the KAT-sized
    two-block model trains and its loss falls."""
    _need(REF_EXE)
    hist = _train(REF_EXE, _model("two_block.json"), 8, 0.2, 16, 128, 4, 8)
    assert len(hist) == 8 and hist[-1][1] < hist[0][1]


@pytest.mark.gpu
@pytest.mark.parametrize("model,batch,spatial", [("two_block.json", 8, 8), ("mobilenet_like.json", 4, 32)])
def test_network_gradients_match_reference(model, batch, spatial):
    _need(REF_EXE)
    _need(GPU_EXE)
    r = _grad(REF_EXE, model, batch, spatial)
    g = _grad(GPU_EXE, model, batch, spatial)
    assert _nrel(g["logits"], r["logits"]) <= 1e-4
    assert abs(g["loss"] - r["loss"]) <= 1e-4 * abs(r["loss"])
    n_scc = 0
    for sg, sr in zip(g["stages"], r["stages"]):
        n_scc += sr["scc"]
        assert _nrel(sg["weight"], sr["weight"]) <= 1e-4
        if sr["bias"]:
            assert _nrel(sg["bias"], sr["bias"]) <= 1e-4
    assert n_scc >= 2
    assert _nrel(g["head_weight"], r["head_weight"]) <= 1e-4


@pytest.mark.gpu
def test_sgd_history_matches_reference():
    """8 epochs of the reference's minibatch SGD (train.cpp) on its synthetic
    dataset: per-epoch loss within 1e-3 relative, same accuracies."""
    _need(REF_EXE)
    _need(GPU_EXE)
    args = (_model("two_block.json"), 8, 0.2, 16, 128, 4, 8)
    r = _train(REF_EXE, *args)
    g = _train(GPU_EXE, *args)
    assert len(r) == len(g) == 8
    for (er, lr, ar), (eg, lg, ag) in zip(r, g):
        assert er == eg
        assert abs(lg - lr) <= 1e-3 * abs(lr), (lg, lr)
        assert abs(ag - ar) <= 1.0 / 128 + 1e-12
