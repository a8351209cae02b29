"""DSX1 fixtures (paper_2101_00745_b200/fixture.py) against the reference's
fixture.cpp, mirroring proj/tests/fixture_test.cpp, and the reference CLI's
golden forward probes (tools/scc/main.cpp:98-132) committed as DSX1 files in
tests/golden/dsx (written by the reference's own fixture_write,
tests/golden/make_dsx.py)."""
import glob
import os
import struct

import numpy as np
import pytest

from conftest import norm_rel

DSX = os.path.join(os.path.dirname(__file__), "golden", "dsx")
PROBES = [(4, 4, 2, "1"), (6, 6, 2, "33%"), (8, 16, 4, "50%"), (12, 12, 3, "2")]


def _fx():
    from paper_2101_00745_b200 import fixture
    return fixture


def test_round_trip_bit_exact(tmp_path):  # fixture_test.cpp:35-52
    fx = _fx()
    t = np.random.default_rng(99).standard_normal((2, 4, 3, 3))
    p, p2 = str(tmp_path / "a.dsx"), str(tmp_path / "b.dsx")
    fx.fixture_write(t, p)
    back = fx.fixture_read(p)
    assert back.shape == t.shape and back.dtype == np.float64
    assert np.array_equal(back.view(np.uint64), t.view(np.uint64))
    fx.fixture_write(back, p2)
    assert open(p, "rb").read() == open(p2, "rb").read()


def test_single_negative_zero(tmp_path):  # fixture_test.cpp:54-62
    fx = _fx()
    p = str(tmp_path / "z.dsx")
    fx.fixture_write(np.full((1, 1, 1, 1), -0.0), p)
    assert np.signbit(fx.fixture_read(p)[0, 0, 0, 0])


def test_bytes_equal_reference_writer(tmp_path, ref):
    """Our writer and the reference's fixture_write produce identical files,
    and each reads the other's."""
    fx = _fx()
    t = np.random.default_rng(3).standard_normal((3, 5, 2, 7))
    mine, theirs = str(tmp_path / "m.dsx"), str(tmp_path / "t.dsx")
    fx.fixture_write(t, mine)
    ref.fixture_write(t, theirs)
    assert open(mine, "rb").read() == open(theirs, "rb").read()
    assert np.array_equal(ref.fixture_read(mine), t) and np.array_equal(fx.fixture_read(theirs), t)


def _bad_files(tmp_path):
    fx = _fx()
    t = np.random.default_rng(5).standard_normal((1, 2, 2, 2))
    good = str(tmp_path / "good.dsx")
    fx.fixture_write(t, good)
    blob = open(good, "rb").read()
    cases = {
        "magic": b"NOPE\0\0\0\0" + b"\0" * 64,            # fixture_test.cpp:64-73
        "truncated": blob[:-8],                            # :75-87
        "trailing": blob + b"x",                           # :89-101
        "zero_extent": b"DSX1" + struct.pack("<4Q", 0, 1, 1, 1),  # :103-116
        "short_header": b"DSX1" + b"\0" * 10,
        "huge_extent": b"DSX1" + struct.pack("<4Q", 1 << 33, 1, 1, 1),
    }
    paths = {}
    for k, v in cases.items():
        paths[k] = str(tmp_path / f"{k}.dsx")
        open(paths[k], "wb").write(v)
    paths["missing"] = str(tmp_path / "nonexistent" / "missing.dsx")  # :118-120
    return paths


def test_rejects_malformed_files(tmp_path):
    fx = _fx()
    for name, p in _bad_files(tmp_path).items():
        with pytest.raises(fx.FormatError):
            fx.fixture_read(p)


def test_rejects_exactly_what_the_reference_rejects(tmp_path, ref):
    from oracle.oracle import OracleError
    for name, p in _bad_files(tmp_path).items():
        with pytest.raises(OracleError) as e:
            ref.fixture_read(p)
        assert e.value.code == 8, name  # sccl::FormatError


def test_golden_dsx_files_are_the_references(tmp_path, ref):
    """Regenerating the probes with the reference reproduces the committed
    files byte for byte (the CLI's own check, main.cpp:118-126)."""
    ref.fixture_probes(str(tmp_path), 1)
    committed = sorted(os.path.basename(p) for p in glob.glob(os.path.join(DSX, "*.dsx")))
    assert len(committed) == 16
    for name in committed:
        assert open(os.path.join(DSX, name), "rb").read() == open(str(tmp_path / name), "rb").read(), name


def test_golden_probes_against_the_oracle(port):
    """The committed probe outputs equal the C port's forward on the committed
    inputs (fp64, bit for bit: the port follows kernel.cpp:45-60's order)."""
    fx = _fx()
    for i, (ci, co, cg, ov) in enumerate(PROBES):
        x = fx.fixture_read(os.path.join(DSX, f"probe_{i}_input.dsx"))
        w = fx.fixture_read(os.path.join(DSX, f"probe_{i}_weight.dsx")).ravel()
        b = fx.fixture_read(os.path.join(DSX, f"probe_{i}_bias.dsx")).ravel()
        y = fx.fixture_read(os.path.join(DSX, f"probe_{i}.dsx"))
        assert x.shape == (2, ci, 5, 5) and y.shape == (2, co, 5, 5)
        ovl = ("ratio", float(ov[:-1]) / 100) if ov.endswith("%") else ("channels", int(ov))
        cfg = port.config(ci, co, cg, ovl, True)
        assert np.array_equal(port.forward(cfg, x, w, b), y)


@pytest.mark.gpu
@pytest.mark.parametrize("path", ["tensor", "cuda_core"])
def test_golden_probes_gpu(path):
    """The GPU forward on the DSX1 probe inputs (fp32) matches the reference's
    golden outputs within the forward bar."""
    import torch
    import paper_2101_00745_b200 as scc
    from paper_2101_00745_b200 import _lib
    fx = _fx()
    for i, (ci, co, cg, ov) in enumerate(PROBES):
        cfg = scc.scc_config_new(ci, co, cg, ov, True)
        cfg.set_path(_lib.SCC_PATH_TENSOR if path == "tensor" else _lib.SCC_PATH_CUDA_CORE)
        x = torch.from_numpy(fx.fixture_read(os.path.join(DSX, f"probe_{i}_input.dsx")).astype(np.float32)).cuda()
        w = torch.from_numpy(fx.fixture_read(os.path.join(DSX, f"probe_{i}_weight.dsx")).ravel().astype(np.float32)).cuda()
        b = torch.from_numpy(fx.fixture_read(os.path.join(DSX, f"probe_{i}_bias.dsx")).ravel().astype(np.float32)).cuda()
        y = scc.scc_forward(x, scc.SccWeights(w, b), cfg)
        # fp32 inputs: the golden is the fp64 forward of the fp64 inputs
        assert norm_rel(y.cpu().numpy(), fx.fixture_read(os.path.join(DSX, f"probe_{i}.dsx"))) <= 1e-5
