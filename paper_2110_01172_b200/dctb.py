"""DCTB tensor files — the container the reference's file front end reads and
writes around the transforms (proj/src/io.cpp:60-107, proj/include/sdct/io.hpp:1-9).

Layout: magic ``b"DCTB"``, one version byte (1), one rank byte (1..4), ``rank``
little-endian uint64 extents, then the row-major payload as little-endian
IEEE-754 doubles. Every structural defect the reference rejects raises
``FormatError`` here too (bad magic, unsupported version, rank outside 1..4,
zero extent, extent product overflowing 64 bits, truncated payload, trailing
bytes, unopenable file); ``write_dctb`` refuses ranks outside 1..4 with
``ShapeError`` (io.cpp:97-99).

``transform_file`` is the file-to-file transform of the reference's
``transform`` subcommand (proj/tools/sdct_main.cpp:67-125): same kind names,
the same rank checks and ``--algo`` / ``--normalize`` semantics, with the
transform itself on the GPU. Reading goes straight from the file into the
array (no per-element decode loop), so a 4096² payload costs one read.
"""
from __future__ import annotations

import os
import struct

import numpy as np

from ._sdct import FormatError, ShapeError

MAGIC = b"DCTB"
VERSION = 1
MAX_RANK = 4
_U64_MAX = (1 << 64) - 1


class UsageError(ValueError):
    """Kind / rank / option misuse (the CLI's exit-code-2 class, sdct_main.cpp:37-41)."""


def _header(dims) -> bytes:
    return MAGIC + bytes([VERSION, len(dims)]) + struct.pack(f"<{len(dims)}Q", *dims)


def read_header(f, path: str):
    """Parse and validate the header at the start of `f`; returns the extents
    (io.cpp:63-85: magic, version, rank, extents, overflow)."""
    magic = f.read(4)
    if len(magic) < 4 or magic != MAGIC:
        raise FormatError(f"DCTB: bad magic in {path}")
    vr = f.read(1)
    if not vr:
        raise FormatError(f"DCTB: truncated header in {path}")
    if vr[0] != VERSION:
        raise FormatError(f"DCTB: unsupported version {vr[0]} in {path}")
    rk = f.read(1)
    if not rk:
        raise FormatError(f"DCTB: truncated header in {path}")
    rank = rk[0]
    if rank < 1 or rank > MAX_RANK:
        raise FormatError(f"DCTB: rank {rank} outside 1..4 in {path}")
    dims, count = [], 1
    for _ in range(rank):
        b = f.read(8)
        if len(b) < 8:
            raise FormatError("DCTB: truncated while reading extents")
        d = struct.unpack("<Q", b)[0]
        if d == 0:
            raise FormatError(f"DCTB: zero extent in {path}")
        if d > _U64_MAX // count:
            raise FormatError(f"DCTB: extents overflow in {path}")
        dims.append(d)
        count *= d
    return tuple(dims)


def read_dctb(path) -> np.ndarray:
    """Read a DCTB file into a float64 array of its shape (sdct::read_dctb)."""
    path = os.fspath(path)
    try:
        f = open(path, "rb")
    except OSError:
        raise FormatError(f"DCTB: cannot open {path}") from None
    with f:
        dims = read_header(f, path)
        count = 1
        for d in dims:
            count *= d
        left = os.fstat(f.fileno()).st_size - f.tell()
        if left < 8 * count:
            raise FormatError("DCTB: truncated while reading payload")
        if left > 8 * count:
            # anything after the payload means the dims lied about the size
            raise FormatError(f"DCTB: trailing bytes after payload in {path}")
        data = np.fromfile(f, dtype="<f8", count=count)
    return data.astype(np.float64, copy=False).reshape(dims)


def write_dctb(path, x) -> None:
    """Write `x` (numpy array or tensor, any real dtype; stored as float64) as
    a DCTB file (sdct::write_dctb)."""
    path = os.fspath(path)
    if hasattr(x, "detach"):  # torch tensor, any device
        x = x.detach().to("cpu").double().numpy()
    a = np.asarray(x, dtype="<f8")
    if a.ndim < 1 or a.ndim > MAX_RANK:
        raise ShapeError(f"DCTB files cover rank 1..4, got rank {a.ndim}")
    a = np.ascontiguousarray(a)
    try:
        with open(path, "wb") as f:
            f.write(_header(a.shape))
            a.tofile(f)
    except OSError as e:
        raise FormatError(f"DCTB: write failed for {path}: {e}") from None


# kind -> (rank, api function name, normalisation factor of the inverse as a
# function of the extents) — sdct_main.cpp:73-113
_KINDS = {
    "dct1": (1, "dct_1d", None),
    "idct1": (1, "idct_1d", lambda d: 2.0 / d[0]),
    "idxst1": (1, "idxst_1d", lambda d: 2.0 / d[0]),
    "dct2": (2, "dct_2d", None),
    "idct2": (2, "idct_2d", lambda d: 4.0 / (d[0] * d[1])),
    "idct-idxst": (2, "idct_idxst_2d", lambda d: 4.0 / (d[0] * d[1])),
    "idxst-idct": (2, "idxst_idct_2d", lambda d: 4.0 / (d[0] * d[1])),
    "dct3": (3, "dct_3d", None),
    "idct3": (3, "idct_3d", lambda d: 8.0 / (d[0] * d[1] * d[2])),
}
_ALGOS = ("4n", "2n-mirrored", "2n-padded", "n")


def transform_file(input_path, output_path, kind: str, algo: str = "n", normalize: bool = False,
                   threads: int = 0) -> np.ndarray:
    """DCTB -> transform on the GPU -> DCTB (the reference's ``sdct transform``).

    ``normalize`` rescales the inverse kinds so that they invert the forward
    ones exactly (2/N, 4/(N1 N2), 8/(N1 N2 N3)); ``algo`` picks the 1D DCT
    variant and is valid only with ``kind="dct1"``. Returns the result."""
    from . import api

    x = read_dctb(input_path)
    if algo != "n" and kind != "dct1":
        raise UsageError("--algo applies only to --kind dct1")
    if kind not in _KINDS:
        raise UsageError(f"unknown --kind '{kind}'")
    rank, fn, norm = _KINDS[kind]
    if x.ndim != rank:
        raise UsageError(f"--kind {kind} needs a rank-{rank} tensor, but the input has rank {x.ndim}")
    if kind == "dct1":
        if algo not in _ALGOS:
            raise UsageError(f"unknown --algo '{algo}' (expected 4n, 2n-mirrored, 2n-padded or n)")
        y = api.dct_1d(x, variant=algo, threads=threads)
    else:
        y = getattr(api, fn)(x, threads=threads)
    if normalize and norm is not None:
        y = y * norm(x.shape)
    write_dctb(output_path, y)
    return y
