"""Write the DCTB fixtures in tests/golden/dctb/ with the UNMODIFIED
reference writer (sdct::write_dctb, proj/src/io.cpp:96-107, called through the
oracle/_ref shim). Run in the build container after `make -C oracle ref`:

    python tests/golden/make_dctb.py

The payloads follow the reference's CLI test fixtures
(proj/tests/cli_tests.sh:57-59) plus one seeded tensor per rank 3 and 4.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402

FIXTURES = {
    "ones2x2": np.ones((2, 2)),
    "vec8": np.array([0.3, -1.2, 2.5, 0.0, 4.1, -0.7, 1.9, 0.25]),
    "grid6x4": np.array([((3 * i) % 7) - 3.0 for i in range(24)]).reshape(6, 4),
    "cube3x4x5": np.random.default_rng(71).uniform(-100.0, 100.0, (3, 4, 5)),
    "rank4_2x2x2x3": np.random.default_rng(72).uniform(-100.0, 100.0, (2, 2, 2, 3)),
}


def main() -> None:
    out = os.path.join(HERE, "dctb")
    os.makedirs(out, exist_ok=True)
    for name, x in FIXTURES.items():
        rc = oracle.ref.write_dctb(os.path.join(out, name + ".dctb"), x)
        assert rc == 0, name
    print("wrote", sorted(FIXTURES))


if __name__ == "__main__":
    main()
