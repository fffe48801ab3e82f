"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Run in the build container (where /root/reference exists):

    make -C oracle ref                 # compiles the reference + its pybind module
    python tests/golden/make_golden.py

The reference's own pybind11 module (proj/bindings/module.cpp, compiled by
oracle/Makefile into oracle/_ref/python/sdct) is imported and called through its
public Python API (`sdct.dct_2d`, ...). Inputs are seeded numpy uniform(-1, 1),
the distribution the reference's tests use (proj/tests/test_dct2d.cpp:17-23,
proj/tests/python/test_smoke.py:14). Outputs are stored as float64.

The fixture files are committed; the GPU box never needs /root/reference.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref", "python"))

import sdct  # noqa: E402  (the reference module)

SHAPES_2D = [(n1, n2) for n1 in range(1, 9) for n2 in range(1, 9)] + [
    (5, 7), (16, 12), (31, 17), (64, 64), (33, 17), (24, 17), (13, 21), (9, 14), (16, 3),
    (3, 16), (2, 64), (64, 2), (32, 32), (128, 128), (128, 64), (64, 256), (100, 60),
]
SHAPES_3D = [(2, 2, 2), (3, 4, 5), (5, 4, 3), (2, 3, 4), (8, 8, 8), (5, 6, 7), (7, 8, 9),
             (16, 16, 16), (4, 8, 16), (16, 8, 4), (32, 32, 32)]
KINDS_2D = ["dct_2d", "idct_2d", "idct_idxst_2d", "idxst_idct_2d", "dct_2d_rowcol"]
KINDS_3D = ["dct_3d", "idct_3d"]


def main() -> None:
    out = {}
    seed = 1000
    for shape in SHAPES_2D:
        seed += 1
        x = np.random.default_rng(seed).uniform(-1.0, 1.0, size=shape)
        key = "x".join(map(str, shape))
        out[f"in/{key}"] = x
        for kind in KINDS_2D:
            out[f"{kind}/{key}"] = getattr(sdct, kind)(x)
        # spectral force fields (proj/src/force.cpp:11-37, module.cpp:163-171)
        xi1, xi2 = sdct.force_demo_fields(x)
        out[f"force_xi1/{key}"] = xi1
        out[f"force_xi2/{key}"] = xi2
    for shape in SHAPES_3D:
        seed += 1
        x = np.random.default_rng(seed).uniform(-1.0, 1.0, size=shape)
        key = "x".join(map(str, shape))
        out[f"in/{key}"] = x
        for kind in KINDS_3D:
            out[f"{kind}/{key}"] = getattr(sdct, kind)(x)
    # rank-4 factorised DCT (transforms_ext.cpp:396-425) and the brute-force
    # cosine-sum oracles the reference module exports (module.cpp:144-158)
    for shape in [(2, 3, 4, 5), (4, 4, 8, 8), (3, 2, 16, 8), (8, 16, 4, 2)]:
        seed += 1
        x = np.random.default_rng(seed).uniform(-1.0, 1.0, size=shape)
        key = "x".join(map(str, shape))
        out[f"in/{key}"] = x
        out[f"dct_4d/{key}"] = sdct.dct_4d(x)
    for n in (1, 5, 16, 37):
        seed += 1
        x = np.random.default_rng(seed).uniform(-1.0, 1.0, size=(n,))
        out[f"in/{n}"] = x
        out[f"dct_oracle_1d/{n}"] = sdct.dct_oracle_1d(x)
    for shape in [(3, 5), (8, 8), (16, 12)]:
        key = "x".join(map(str, shape))
        out[f"dct_oracle_2d/{key}"] = sdct.dct_oracle_2d(out[f"in/{key}"])
    # Known-answer inputs (proj/tests/cli_tests.sh:113-121,
    # proj/tests/test_transforms_ext.cpp:180-185).
    out["kat/ones2x2/in"] = np.ones((2, 2))
    out["kat/ones2x2/dct_2d"] = sdct.dct_2d(np.ones((2, 2)))
    delta = np.zeros((2, 2))
    delta[0, 0] = 1.0
    out["kat/delta2x2/in"] = delta
    out["kat/delta2x2/dct_2d"] = sdct.dct_2d(delta)
    out["kat/ones2x2x2/in"] = np.ones((2, 2, 2))
    out["kat/ones2x2x2/dct_3d"] = sdct.dct_3d(np.ones((2, 2, 2)))
    path = os.path.join(HERE, "golden_ref.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(out)} arrays, {os.path.getsize(path) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
