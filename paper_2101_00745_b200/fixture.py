"""DSX1 tensor fixtures: the reference's golden-file format
(proj/core/src/fixture.cpp:29-97, fixture.hpp:9-19).

Layout: the 4-byte tag ``DSX1``, four little-endian uint64 extents (n, c, h,
w), then n*c*h*w IEEE-754 float64 values, little-endian, row-major (NCHW).
Round trips are bit exact.  ``fixture_read`` raises ``FormatError`` on a
missing file, a bad tag, zero / oversized extents, a truncated payload or
trailing bytes -- the checks of fixture.cpp:59-85, in the same order.
"""
from __future__ import annotations

import numpy as np

from ._lib import SccError

_MAGIC = b"DSX1"
_MAX_ELEMENTS = 1 << 32  # fixture.cpp:72


class FormatError(SccError):
    """sccl::FormatError (errors.hpp:38-42): a malformed fixture file."""

    code = 8


def fixture_write(t, path: str) -> None:
    """fixture_write (fixture.cpp:29-50): any 4-d array-like (float64 on disk)."""
    a = np.ascontiguousarray(np.asarray(t, dtype=np.float64))
    if a.ndim != 4:
        raise FormatError(f"fixture tensors are 4-d (NCHW), got {a.ndim}-d")
    try:
        with open(path, "wb") as f:
            f.write(_MAGIC)
            f.write(np.asarray(a.shape, dtype="<u8").tobytes())
            f.write(a.astype("<f8", copy=False).tobytes())
    except OSError as e:
        raise FormatError(f"cannot open '{path}' for writing") from e


def fixture_read(path: str) -> np.ndarray:
    """fixture_read (fixture.cpp:52-95) -> float64 array [n, c, h, w]."""
    try:
        with open(path, "rb") as f:
            blob = f.read()
    except OSError as e:
        raise FormatError(f"cannot open '{path}' for reading") from e
    if len(blob) < 36:
        raise FormatError(f"'{path}': truncated header")
    if blob[:4] != _MAGIC:
        raise FormatError(f"'{path}': bad magic tag")
    ext = [int(v) for v in np.frombuffer(blob, dtype="<u8", count=4, offset=4)]
    count = 1
    for e in ext:
        if e == 0 or e > _MAX_ELEMENTS or count > _MAX_ELEMENTS // e:
            raise FormatError(f"'{path}': nonsensical extents in header")
        count *= e
    payload = len(blob) - 36
    if payload < 8 * count:
        raise FormatError(f"'{path}': payload shorter than extents imply")
    if payload > 8 * count:
        raise FormatError(f"'{path}': trailing bytes after payload")
    return np.frombuffer(blob, dtype="<f8", count=count, offset=36).astype(np.float64).reshape(ext)
