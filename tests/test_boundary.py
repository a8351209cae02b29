"""CPU tests of the drop-in boundary (no GPU needed).

* libscc_b200.so loads and exports every symbol include/scc_b200.h declares.
* The host geometry behind the C ABI (Overlap parse/resolve, scc_config_new,
  compute_channel_cycle, window_of, covering_filters, MAC count) agrees
  exactly with the compiled reference, including its error classes.
* Device entry points fail loudly (status SCC_ERR_CUDA, never a CPU result)
  when no sm_100 device is present.
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2101_00745_b200 as scc
from paper_2101_00745_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "scc_b200.h")


def test_library_exports_every_declared_symbol():
    src = open(HEADER).read()
    declared = set(re.findall(
        r"^\s*(?:scc_status_t|const char\*|int|uint64_t)\s+(scc_\w+)\s*\(", src, re.M))
    assert declared == set(_lib.EXPORTS), declared ^ set(_lib.EXPORTS)
    L = _lib.lib()
    for name in declared:
        assert hasattr(L, name), name
    assert L.scc_abi_version() == 1


def test_overlap_text_forms(ref):  # config_test.cpp:9-19
    for text, gw, want in [("50%", 2, 1), ("0.5", 2, 1), ("3", 8, 3), ("0", 8, 0),
                           ("33%", 3, 1), ("100%", 4, 4), ("70%", 8, 6), ("1e-1", 10, 1)]:
        assert scc.Overlap.parse(text).resolve(gw) == want == ref.resolve(text, gw)
    for bad in ("abc", "", "12x", "5%%", "1.5.2"):
        with pytest.raises(scc.ArgumentError):
            scc.Overlap.parse(bad)


def test_overlap_range(ref):  # config_test.cpp:21-28
    with pytest.raises(scc.ConfigError):
        scc.Overlap.ratio(1.5).resolve(4)
    with pytest.raises(scc.ConfigError):
        scc.Overlap.ratio(-0.1).resolve(4)
    with pytest.raises(scc.ConfigError):
        scc.Overlap.channels(5).resolve(4)
    with pytest.raises(scc.ConfigError):
        scc.Overlap.channels(-1).resolve(4)
    assert scc.Overlap.ratio(1.0).resolve(4) == 4
    assert scc.Overlap.ratio(0.0).resolve(4) == 0
    assert scc.Overlap.ratio(0.5).str() == "50%"
    assert scc.Overlap.channels(2).str() == "2"


def test_llround_half_away_from_zero(ref):
    # config.cpp:45 -- Python's round(2.5) would give 2.
    for gw in range(1, 40):
        for pct in (25, 50, 75, 33, 70, 12.5):
            assert scc.Overlap.ratio(pct / 100).resolve(gw) == ref.resolve(("ratio", pct / 100), gw)


def test_config_validation():  # config_test.cpp:53-66
    for args in [(4, 4, 3, "0"), (4, 4, 2, "3"), (0, 4, 1, "0"), (4, 0, 2, "0"),
                 (4, 4, 0, "0"), (4, 4, 8, "0")]:
        with pytest.raises(scc.ConfigError):
            scc.scc_config_new(*args, True)


def test_fully_overlapped():  # config_test.cpp:68-79
    assert scc.scc_config_new(4, 4, 2, scc.Overlap.channels(2), True).fully_overlapped()
    assert not scc.scc_config_new(4, 4, 1, scc.Overlap.ratio(1.0), True).fully_overlapped()
    assert not scc.scc_config_new(4, 4, 2, scc.Overlap.channels(1), True).fully_overlapped()


def test_window_lookup():  # cycle_test.cpp:55-67
    cfg = scc.scc_config_new(4, 4, 2, scc.Overlap.channels(1), True)
    cyc = scc.compute_channel_cycle(cfg)
    w3 = scc.window_of(cyc, 3)
    assert w3.start == 3 and w3.contains(3, 4) and w3.contains(0, 4) and not w3.contains(1, 4)
    assert w3.last(4) == 0
    assert scc.window_of(cyc, 7) == w3 and scc.window_of(cyc, 0).start == 0
    with pytest.raises(scc.IndexError):
        scc.window_of(cyc, -1)
    # the native lookup agrees and raises the same class
    s, n = C.c_int64(), C.c_int64()
    _lib.check(_lib.lib().scc_plan_window_of(cfg.handle, 7, C.byref(s), C.byref(n)))
    assert (s.value, n.value) == (3, 2)
    with pytest.raises(scc.IndexError):
        _lib.check(_lib.lib().scc_plan_window_of(cfg.handle, -1, C.byref(s), C.byref(n)))


def test_covering_errors():  # cycle_test.cpp:86-87
    cfg = scc.scc_config_new(4, 4, 2, scc.Overlap.channels(1), True)
    with pytest.raises(scc.IndexError):
        scc.covering_filters(cfg, None, 4)
    with pytest.raises(scc.IndexError):
        scc.covering_filters(cfg, None, -1)


def test_geometry_sweep_matches_reference(ref):
    """Every config of the cycle-law sweep (cycle_test.cpp:90-138), both
    Co in {Ci, 2Ci} and a ragged Co: cycle, window starts and covering lists
    equal the reference's exactly."""
    for c_in in (2, 4, 6, 8, 12, 16):
        for cg in [d for d in range(1, c_in + 1) if c_in % d == 0]:
            gw = c_in // cg
            for ov in range(gw + 1):
                for c_out in (c_in, 2 * c_in, c_in + 3):
                    mine = scc.scc_config_new(c_in, c_out, cg, scc.Overlap.channels(ov), True)
                    theirs = ref.config(c_in, c_out, cg, ("channels", ov), True)
                    assert (mine.group_width, mine.overlap_channels, mine.shift) == (
                        theirs.group_width, theirs.overlap_channels, theirs.shift)
                    cyc = scc.compute_channel_cycle(mine)
                    assert [w.start for w in cyc.windows] == ref.cycle(theirs)
                    for oc in range(c_out + 5):
                        assert scc.window_of(cyc, oc).start == ref.window_of(theirs, oc)
                    for ic in range(c_in):
                        assert scc.covering_filters(mine, cyc, ic) == ref.covering(theirs, ic)


def test_baseline_geometries_match_reference(ref):
    """The BASELINE shapes (config 1 and the cg x co x C sweep)."""
    shapes = [(64, 128, 2, "50%")]
    for c in (256, 512, 1024):
        for cg in (2, 4, 8):
            for co in ("25%", "50%", "75%"):
                shapes.append((c, c, cg, co))
    for c_in, c_out, cg, co in shapes:
        mine = scc.scc_config_new(c_in, c_out, cg, co, True)
        theirs = ref.config(c_in, c_out, cg, co, True)
        assert (mine.overlap_channels, mine.shift) == (theirs.overlap_channels, theirs.shift)
        assert [w.start for w in scc.compute_channel_cycle(mine).windows] == ref.cycle(theirs)
        for ic in (0, 1, c_in // 2, c_in - 1):
            assert scc.covering_filters(mine, None, ic) == ref.covering(theirs, ic)


def test_mac_count():  # kernel_test.cpp:255-265
    cfg = scc.scc_config_new(8, 12, 4, scc.Overlap.channels(1), True)
    assert scc.scc_forward_macs(cfg, 2, 3, 5) == 2 * 12 * 3 * 5 * cfg.group_width


def test_device_entry_points_fail_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by the gpu suite")
    cfg = scc.scc_config_new(8, 8, 2, "50%", True)
    rc = _lib.lib().scc_forward_f32(cfg.handle, 1, 2, 2, 16, 16, 16, 16, None)
    assert rc == _lib.SCC_ERR_CUDA
    assert "sm_100" in _lib.lib().scc_last_error().decode() or "CUDA" in \
        _lib.lib().scc_last_error().decode() or "cuda" in _lib.lib().scc_last_error().decode()


def test_argument_checks_precede_device_work():
    cfg = scc.scc_config_new(8, 8, 2, "50%", True)
    L = _lib.lib()
    # zero extents -> ShapeError (Tensor4 requires extents >= 1, tensor.cpp:11-18)
    assert L.scc_forward_f32(cfg.handle, 0, 2, 2, 16, 16, 16, 16, None) == _lib.SCC_ERR_SHAPE
    # missing bias on a biased layer -> ShapeError (check_weights, kernel.cpp:20-24)
    assert L.scc_forward_f32(cfg.handle, 1, 2, 2, 16, 16, None, 16, None) == _lib.SCC_ERR_SHAPE
    # null input -> ArgumentError
    assert L.scc_forward_f32(cfg.handle, 1, 2, 2, None, 16, 16, 16, None) == _lib.SCC_ERR_ARGUMENT
    nb = scc.scc_config_new(8, 8, 2, "50%", False)
    assert L.scc_forward_f32(nb.handle, 1, 2, 2, 16, 16, 16, 16, None) == _lib.SCC_ERR_SHAPE


def test_workspace_size_is_host_only():
    cfg = scc.scc_config_new(64, 128, 2, "50%", True)
    assert cfg.workspace_bytes(32, 32, 32) > 0
    cfg2 = scc.scc_config_new(1024, 1024, 2, "50%", True)
    assert cfg2.workspace_bytes(32, 56, 56) < 512 << 20
