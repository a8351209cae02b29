"""Pin the CPU oracle (oracle/scc_oracle.c) before trusting it.

1. The reference's own known-answer tests (proj/tests/kernel_test.cpp,
   cycle_test.cpp, config_test.cpp) re-expressed against both the C port and
   the compiled reference.
2. Port == compiled reference, bit for bit, on random geometries.
3. Port == golden fixtures (generated from the compiled reference by
   tests/golden/make_golden.py), bit for bit.
"""
import glob
import math
import os

import numpy as np
import pytest

from conftest import norm_rel

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "probe_*.npz")))


def _oracles(port, ref_or_none):
    return [port] + ([ref_or_none] if ref_or_none is not None else [])


@pytest.fixture(scope="module")
def both(port):
    from oracle import load_ref
    return _oracles(port, load_ref())


def col(vals):
    return np.array(vals, np.float64).reshape(1, len(vals), 1, 1)


def test_forward_worked_example(both):  # kernel_test.cpp:33-43
    for o in both:
        cfg = o.config(4, 4, 2, ("channels", 1), False)
        y = o.forward(cfg, col([1, 2, 3, 4]), np.ones(8), None)
        assert list(y.ravel()) == [3.0, 5.0, 7.0, 5.0]


def test_bias_only_forward(both):  # kernel_test.cpp:45-63
    rng = np.random.default_rng(2)
    for o in both:
        cfg = o.config(6, 6, 3, ("channels", 0), True)
        x = rng.standard_normal((2, 6, 3, 2))
        y = o.forward(cfg, x, np.zeros(6 * 2), np.arange(6.0))
        for oc in range(6):
            assert np.all(y[:, oc] == oc)


def test_backward_input_worked_example(both):  # kernel_test.cpp:65-71
    for o in both:
        cfg = o.config(4, 4, 2, ("channels", 1), False)
        dx = o.backward_input(cfg, np.ones((1, 4, 1, 1)), np.ones(8))
        assert list(dx.ravel()) == [2.0] * 4


def test_backward_params_worked_example(both):  # kernel_test.cpp:73-83
    for o in both:
        cfg = o.config(4, 4, 2, ("channels", 1), False)
        dw, _ = o.backward_params(cfg, np.ones((1, 4, 1, 1)), col([1, 2, 3, 4]))
        assert dw[0 * 2 + 0] == 1.0 and dw[0 * 2 + 1] == 2.0
        assert dw[3 * 2 + 0] == 4.0 and dw[3 * 2 + 1] == 1.0


def test_bias_gradient(both):  # kernel_test.cpp:85-93
    for o in both:
        cfg = o.config(4, 4, 2, ("channels", 1), True)
        _, db = o.backward_params(cfg, np.ones((1, 4, 2, 2)), np.full((1, 4, 2, 2), 0.5))
        assert list(db) == [4.0] * 4


def test_zero_cotangent(both):  # kernel_test.cpp:95-106
    rng = np.random.default_rng(4)
    for o in both:
        cfg = o.config(8, 8, 4, ("channels", 1), True)
        x = rng.standard_normal((2, 8, 3, 3))
        w = rng.uniform(-0.5, 0.5, 16)
        g = np.zeros((2, 8, 3, 3))
        assert np.all(o.backward_input(cfg, g, w) == 0)
        dw, db = o.backward_params(cfg, g, x)
        assert np.all(dw == 0) and np.all(db == 0)


def test_cycle_examples(both):  # cycle_test.cpp:32-53
    for o in both:
        assert o.cycle(o.config(4, 4, 2, ("ratio", 0.5))) == [0, 1, 2, 3]
        assert o.cycle(o.config(6, 6, 2, ("ratio", 0.33))) == [0, 2, 4]
        assert len(o.cycle(o.config(4, 4, 2, ("channels", 2)))) == 1
        assert o.cycle(o.config(8, 4, 8, ("channels", 0))) == [0, 1, 2, 3]


def test_covering_examples(both):  # cycle_test.cpp:69-88
    for o in both:
        a = o.config(4, 4, 2, ("channels", 1))
        assert o.covering(a, 1) == [0, 1]
        wide = o.config(4, 8, 2, ("channels", 1))
        assert o.covering(wide, 3) == [2, 3, 6, 7]
        dense = o.config(4, 5, 1, ("ratio", 0.5))
        for ic in range(4):
            assert o.covering(dense, ic) == [0, 1, 2, 3, 4]


def test_fan_in_nonuniform(port):
    cfg = port.config(8, 5, 4, ("channels", 1))
    assert [len(port.covering(cfg, ic)) for ic in range(8)] == [1, 2, 2, 2, 2, 1, 0, 0]
    cfg = port.config(6, 4, 2, ("channels", 1))
    assert [len(port.covering(cfg, ic)) for ic in range(6)] == [3, 2, 3, 1, 2, 1]


def test_cycle_law_sweep(both):  # cycle_test.cpp:90-111, acceptance.cpp:208-259
    for o in both:
        for c_in in (2, 4, 6, 8, 12, 16):
            for cg in [d for d in range(1, c_in + 1) if c_in % d == 0]:
                gw = c_in // cg
                for ov in range(gw + 1):
                    for c_out in (c_in, 2 * c_in):
                        cfg = o.config(c_in, c_out, cg, ("channels", ov))
                        starts = o.cycle(cfg)
                        shift = gw - ov
                        period = 1 if shift == 0 else c_in // math.gcd(shift, c_in)
                        assert len(starts) == min(c_out, period)
                        for oc in range(c_out):
                            assert starts[oc % len(starts)] == (oc * shift) % c_in


def test_config_resolution(ref):  # config_test.cpp:9-51
    assert ref.resolve("50%", 2) == 1
    assert ref.resolve("0.5", 2) == 1
    assert ref.resolve("3", 8) == 3
    assert ref.resolve("33%", 3) == 1
    assert ref.resolve("100%", 4) == 4
    c = ref.config(8, 16, 1, "70%", False)
    assert (c.group_width, c.overlap_channels, c.shift, c.has_bias) == (8, 6, 2, False)
    # llround: halves away from zero (config.cpp:45) -- gw=5 at 50% is 3.
    assert ref.resolve(("ratio", 0.5), 5) == 3


def test_port_equals_reference_bitwise(port, ref):
    rng = np.random.default_rng(7)
    for trial in range(25):
        c_in = int(rng.integers(1, 13)) * 2
        divs = [d for d in range(1, c_in + 1) if c_in % d == 0]
        cg = int(rng.choice(divs))
        gw = c_in // cg
        ov = int(rng.integers(0, gw + 1))
        c_out = int(rng.integers(1, 2 * c_in + 1))
        hb = bool(rng.integers(0, 2))
        cfg_p = port.config(c_in, c_out, cg, ("channels", ov), hb)
        cfg_r = ref.config(c_in, c_out, cg, ("channels", ov), hb)
        assert cfg_p == cfg_r
        n, h, w = int(rng.integers(1, 4)), int(rng.integers(1, 6)), int(rng.integers(1, 6))
        x = rng.standard_normal((n, c_in, h, w)).astype(np.float32)
        wt = rng.uniform(-1, 1, c_out * gw).astype(np.float32)
        b = rng.uniform(-0.5, 0.5, c_out).astype(np.float32) if hb else None
        dy = rng.standard_normal((n, c_out, h, w)).astype(np.float32)
        assert np.array_equal(port.forward(cfg_p, x, wt, b), ref.forward(cfg_r, x, wt, b))
        assert np.array_equal(port.backward_input(cfg_p, dy, wt), ref.backward_input(cfg_r, dy, wt))
        dwp, dbp = port.backward_params(cfg_p, dy, x)
        dwr, dbr = ref.backward_params(cfg_r, dy, x)
        assert np.array_equal(dwp, dwr)
        if hb:
            assert np.array_equal(dbp, dbr)
        for ic in range(c_in):
            assert port.covering(cfg_p, ic) == ref.covering(cfg_r, ic)


@pytest.mark.parametrize("path", GOLDEN, ids=lambda p: os.path.basename(p))
def test_port_matches_golden(port, path):
    g = np.load(path)
    ci, co, cg, hb, n, h, w = (int(v) for v in g["geometry"])
    cfg = port.config(ci, co, cg, ("channels", int(g["cfg"][0])), bool(hb))
    assert [cfg.overlap_channels, cfg.group_width, cfg.shift] == list(g["cfg"])
    assert port.cycle(cfg) == list(g["starts"])
    b = g["b"] if hb else None
    assert np.array_equal(port.forward(cfg, g["x"], g["w"], b), g["y"])
    assert np.array_equal(port.backward_input(cfg, g["dy"], g["w"]), g["dx"])
    dw, db = port.backward_params(cfg, g["dy"], g["x"])
    assert np.array_equal(dw, g["dw"])
    if hb:
        assert np.array_equal(db, g["db"])


def test_adjoint_identity_port(port):  # kernel_test.cpp:172-207
    rng = np.random.default_rng(55)
    for _ in range(10):
        c_in = 2 * int(rng.integers(1, 7))
        divs = [d for d in range(1, c_in + 1) if c_in % d == 0]
        cg = int(rng.choice(divs))
        gw = c_in // cg
        cfg = port.config(c_in, int(rng.integers(1, 2 * c_in + 1)), cg,
                          ("channels", int(rng.integers(0, gw + 1))), False)
        w = rng.uniform(-1, 1, cfg.c_out * gw)
        x = rng.standard_normal((2, c_in, 3, 3))
        g = rng.standard_normal((2, cfg.c_out, 3, 3))
        lhs = float(np.sum(g * port.forward(cfg, x, w, None)))
        rhs = float(np.sum(port.backward_input(cfg, g, w) * x))
        assert norm_rel(lhs, rhs) < 1e-10


@pytest.mark.parametrize("shape", [(2, 5, 7, 6, 3, 1), (1, 8, 8, 8, 3, 2), (3, 4, 9, 5, 3, 2),
                                   (1, 3, 1, 1, 3, 1), (2, 6, 4, 4, 1, 1)])
@pytest.mark.parametrize("with_bias", [True, False])
def test_dw_port_matches_compiled_reference(port, ref, shape, with_bias):
    """The depthwise stage of a dsc_block: the C restatement equals the
    reference's grouped_conv_forward bit for bit (padding, stride 2, 1x1
    planes, kernel 1)."""
    n, c, h, w, k, s = shape
    rng = np.random.default_rng(7)
    x = rng.standard_normal((n, c, h, w))
    wt = rng.uniform(-1, 1, (c, k, k))
    b = rng.uniform(-0.5, 0.5, c) if with_bias else None
    assert np.array_equal(port.dw_forward(x, wt, b, k, s), ref.dw_forward(x, wt, b, k, s))


def test_dw_port_known_answer(port):
    """All-ones 3x3 depthwise on a 3x3 plane of ones: interior 9, edges 6,
    corners 4 (zero padding counts as explicit zeros, reference.cpp:67-72)."""
    y = port.dw_forward(np.ones((1, 1, 3, 3)), np.ones((1, 3, 3)), None)
    assert y[0, 0].tolist() == [[4, 6, 4], [6, 9, 6], [4, 6, 4]]


def test_fp64_class_gemm_reference_matches_oracle(port):
    """tests/fp64_ref.py (the full-batch checker of the GPU sweep parity test)
    equals the oracle to fp64 round-off on random geometries, including
    wrap-around windows, ragged c_out, cg=1, ov=0 and uncovered channels."""
    import torch
    from fp64_ref import scc_fp64
    from conftest import norm_rel
    rng = np.random.default_rng(21)
    cases = [(64, 128, 2, 16), (24, 40, 3, 2), (8, 5, 4, 1), (12, 12, 1, 5), (16, 20, 4, 0),
             (32, 48, 8, 3), (60, 64, 3, 15)]
    for ci, co, cg, ov in cases:
        o = port.config(ci, co, cg, ("channels", ov), True)
        gw = ci // cg
        shift = gw - ov
        x = rng.standard_normal((3, ci, 5, 4))
        dy = rng.standard_normal((3, co, 5, 4))
        w = rng.uniform(-1, 1, co * gw)
        b = rng.uniform(-0.5, 0.5, co)
        y, dx, dw, db = scc_fp64(ci, co, gw, shift, torch.from_numpy(x), torch.from_numpy(w),
                                 torch.from_numpy(b), torch.from_numpy(dy))
        assert norm_rel(y.numpy(), port.forward(o, x, w, b)) <= 1e-13
        assert norm_rel(dx.numpy(), port.backward_input(o, dy, w)) <= 1e-13
        rdw, rdb = port.backward_params(o, dy, x)
        assert norm_rel(dw.numpy(), rdw) <= 1e-13 and norm_rel(db.numpy(), rdb) <= 1e-13
