"""B200-native multi-dimensional DCT library (arXiv 2110.01172, sm_100a).

Drop-in for the reference's ``sdct`` Python module (proj/python/sdct/__init__.py):
the same names, keyword arguments and unnormalised conventions
(``idct_2d(dct_2d(x)) == N1*N2/4 * x``, ``idct_3d(dct_3d(x)) == N1*N2*N3/8 * x``).

* numpy input  -> float64 numpy output (host copies, like the reference);
* torch CUDA tensor input (float32 / float64, optional leading batch dims)
  -> tensor of the same dtype on the same device, no host copies,
  stream-ordered on ``torch.cuda.current_stream()``.

Everything runs on the GPU through ``lib/libsdct_b200.so``. If the native
library is missing or no CUDA device is present, calls raise — there is no
CPU fallback.
"""
from __future__ import annotations

from . import _sdct  # noqa: F401  (raises ImportError when not built)
from ._sdct import DeviceError, FormatError, ShapeError, amdahl_speedup
from .api import (
    compress,
    dct_1d,
    dct_2d,
    dct_2d_rowcol,
    dct_3d,
    dct_4d,
    dct_axis0,
    dct_oracle_1d,
    dct_oracle_2d,
    force_demo_fields,
    idct_1d,
    idct_2d,
    idct_3d,
    idct_axis0,
    idct_idxst_2d,
    idct_idxst_2d_rowcol,
    idxst_1d,
    idxst_idct_2d,
    idxst_idct_2d_rowcol,
    plan_for,
    stream_host,
)
from .dctb import read_dctb, transform_file, write_dctb

__all__ = [
    "ShapeError", "FormatError", "DeviceError", "amdahl_speedup",
    "dct_1d", "idct_1d", "idxst_1d",
    "dct_2d", "dct_2d_rowcol", "idct_2d", "idct_idxst_2d", "idxst_idct_2d",
    "idct_idxst_2d_rowcol", "idxst_idct_2d_rowcol",
    "dct_3d", "dct_4d", "idct_3d", "plan_for", "stream_host", "force_demo_fields",
    "dct_oracle_1d", "dct_oracle_2d", "compress", "dct_axis0", "idct_axis0",
    "read_dctb", "write_dctb", "transform_file",
]

__version__ = "0.1.0"
