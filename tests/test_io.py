"""DCTB tensor files (proj/src/io.cpp:60-107): the Python reader/writer
(paper_2110_01172_b200/dctb.py) and the header-only C++ one (include/sdct/io.hpp)
against the reference's own writer output (tests/golden/dctb/, made by
tests/golden/make_dctb.py with the unmodified reference) and the reference's
defect cases (proj/tests/test_io.cpp:55-125), plus the GPU file-to-file
transform of the reference's `transform` subcommand (proj/tools/sdct_main.cpp:67-125,
proj/tests/cli_tests.sh:104-125)."""
import os
import shutil
import struct
import subprocess

import numpy as np
import pytest

import oracle
from paper_2110_01172_b200 import FormatError, ShapeError
from paper_2110_01172_b200 import dctb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FIX = os.path.join(ROOT, "tests", "golden", "dctb")

# the payloads tests/golden/make_dctb.py wrote through the reference writer
EXPECTED = {
    "ones2x2": np.ones((2, 2)),
    "vec8": np.array([0.3, -1.2, 2.5, 0.0, 4.1, -0.7, 1.9, 0.25]),
    "grid6x4": np.array([((3 * i) % 7) - 3.0 for i in range(24)]).reshape(6, 4),
    "cube3x4x5": np.random.default_rng(71).uniform(-100.0, 100.0, (3, 4, 5)),
    "rank4_2x2x2x3": np.random.default_rng(72).uniform(-100.0, 100.0, (2, 2, 2, 3)),
}


def _header(version, rank, dims, magic=b"DCTB"):
    return magic + bytes([version, rank]) + b"".join(struct.pack("<Q", d) for d in dims)


def _f64(*v):
    return b"".join(struct.pack("<d", x) for x in v)


# proj/tests/test_io.cpp:70-115 — every structural defect is a FormatError
DEFECTS = {
    "bad_magic": b"X" + _header(1, 1, [1])[1:] + _f64(1.0),
    "unsupported_version": _header(2, 1, [1]) + _f64(1.0),
    "rank_zero": _header(1, 0, []),
    "rank_five": _header(1, 5, [1, 1, 1, 1, 1]),
    "zero_extent": _header(1, 2, [3, 0]),
    "truncated_payload": _header(1, 1, [3]) + _f64(1.0),
    "trailing_bytes": _header(1, 1, [1]) + _f64(1.0) + b"\0",
    "extent_overflow": _header(1, 2, [2**64 - 1, 2**64 - 1]),
    "truncated_header": b"DCTB\x01",
    "truncated_extents": _header(1, 2, [3])[:-3],
    "empty_file": b"",
}


@pytest.mark.parametrize("name", sorted(EXPECTED))
def test_reads_reference_written_files(name):
    got = dctb.read_dctb(os.path.join(FIX, name + ".dctb"))
    assert got.dtype == np.float64 and got.shape == EXPECTED[name].shape
    assert np.array_equal(got, EXPECTED[name])  # bit-exact


@pytest.mark.parametrize("name", sorted(EXPECTED))
def test_writes_byte_identical_files(name, tmp_path):
    p = tmp_path / "out.dctb"
    dctb.write_dctb(p, EXPECTED[name])
    assert p.read_bytes() == open(os.path.join(FIX, name + ".dctb"), "rb").read()


def test_round_trips_every_rank_exactly(tmp_path):
    # proj/tests/test_io.cpp:55-68
    rng = np.random.default_rng(7)
    for dims in [(5,), (3, 4), (2, 3, 4), (2, 2, 2, 3)]:
        x = rng.uniform(-100.0, 100.0, dims)
        p = tmp_path / "rt.dctb"
        dctb.write_dctb(p, x)
        back = dctb.read_dctb(p)
        assert back.shape == dims and np.array_equal(back, x)


def test_writer_casts_and_accepts_tensors(tmp_path):
    import torch

    x = torch.arange(12, dtype=torch.float32).reshape(3, 4)
    dctb.write_dctb(tmp_path / "t.dctb", x)
    assert np.array_equal(dctb.read_dctb(tmp_path / "t.dctb"), x.double().numpy())


@pytest.mark.parametrize("name", sorted(DEFECTS))
def test_rejects_structural_defects(name, tmp_path):
    p = tmp_path / f"{name}.dctb"
    p.write_bytes(DEFECTS[name])
    with pytest.raises(FormatError):
        dctb.read_dctb(p)
    if oracle.ref_available():  # the reference rejects the same file
        rc, _ = oracle.ref.read_dctb(str(p))
        assert rc == 3


def test_missing_file_and_rank_errors(tmp_path):
    with pytest.raises(FormatError):
        dctb.read_dctb(tmp_path / "nope.dctb")
    # proj/tests/test_io.cpp:118-121: ranks outside 1..4 are a ShapeError at the API
    with pytest.raises(ShapeError):
        dctb.write_dctb(tmp_path / "r0.dctb", np.float64(1.0))
    with pytest.raises(ShapeError):
        dctb.write_dctb(tmp_path / "r5.dctb", np.zeros((1, 1, 1, 1, 2)))
    assert issubclass(FormatError, ValueError)  # proj/bindings/module.cpp:65


@pytest.mark.skipif(not oracle.ref_available(), reason="reference not built here")
def test_reference_reads_our_files(tmp_path):
    x = np.random.default_rng(3).uniform(-1, 1, (4, 5, 6))
    p = tmp_path / "ours.dctb"
    dctb.write_dctb(p, x)
    rc, back = oracle.ref.read_dctb(str(p))
    assert rc == 0 and np.array_equal(back, x)


CPP = r"""
#include <cstdio>
#include "sdct/io.hpp"
int main(int argc, char** argv) {
  // argv[1]: reference-written grid6x4, argv[2]: output path, argv[3]: defect file
  sdct::RealTensor g = sdct::read_dctb(argv[1]);
  if (g.rank() != 2 || g.dim(0) != 6 || g.dim(1) != 4) return 2;
  for (std::size_t i = 0; i < g.size(); ++i)
    if (g[i] != double((3 * i) % 7) - 3.0) return 3;
  sdct::write_dctb(argv[2], g);
  try { sdct::read_dctb(argv[3]); return 4; } catch (const sdct::FormatError&) {}
  try { sdct::write_dctb(argv[2] + std::string(".r0"), sdct::RealTensor{}); return 5; }
  catch (const sdct::ShapeError&) {}
  std::puts("ok");
  return 0;
}
"""


@pytest.mark.skipif(shutil.which("g++") is None, reason="no host C++ compiler")
def test_cpp_header_matches_reference_files(tmp_path):
    src = tmp_path / "io_check.cpp"
    src.write_text(CPP)
    exe = tmp_path / "io_check"
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)],
                   check=True)
    bad = tmp_path / "bad.dctb"
    bad.write_bytes(DEFECTS["trailing_bytes"])
    out = tmp_path / "cpp.dctb"
    r = subprocess.run([str(exe), os.path.join(FIX, "grid6x4.dctb"), str(out), str(bad)], capture_output=True,
                       text=True)
    assert r.returncode == 0 and r.stdout.strip() == "ok", (r.returncode, r.stdout, r.stderr)
    assert out.read_bytes() == open(os.path.join(FIX, "grid6x4.dctb"), "rb").read()


def test_transform_usage_errors(tmp_path):
    # proj/tests/cli_tests.sh:104-108 — raised before any device work
    src = os.path.join(FIX, "ones2x2.dctb")
    out = tmp_path / "o.dctb"
    with pytest.raises(dctb.UsageError):
        dctb.transform_file(src, out, "dct9")
    with pytest.raises(dctb.UsageError):
        dctb.transform_file(src, out, "dct3")  # rank mismatch
    with pytest.raises(dctb.UsageError):
        dctb.transform_file(src, out, "dct2", algo="4n")
    bad = tmp_path / "badmagic.dctb"
    bad.write_bytes(DEFECTS["bad_magic"])
    with pytest.raises(FormatError):
        dctb.transform_file(bad, out, "dct2")
    assert not out.exists()


@pytest.mark.gpu
def test_transform_file_on_gpu(tmp_path, cuda):
    # proj/tests/cli_tests.sh:113-125: ones -> [[4,0],[0,0]]; dct2 then
    # normalised idct2 returns the input to 1e-10
    flat = tmp_path / "flat.dctb"
    dctb.transform_file(os.path.join(FIX, "ones2x2.dctb"), flat, "dct2")
    assert np.allclose(dctb.read_dctb(flat), [[4.0, 0.0], [0.0, 0.0]], atol=1e-14)
    fwd, back = tmp_path / "fwd.dctb", tmp_path / "back.dctb"
    dctb.transform_file(os.path.join(FIX, "grid6x4.dctb"), fwd, "dct2")
    dctb.transform_file(fwd, back, "idct2", normalize=True)
    assert np.max(np.abs(dctb.read_dctb(back) - EXPECTED["grid6x4"])) < 1e-10
    # every kind against the oracle port on the same file payloads
    cases = {"dct1": "vec8", "idct1": "vec8", "idxst1": "vec8", "dct2": "grid6x4", "idct2": "grid6x4",
             "idct-idxst": "grid6x4", "idxst-idct": "grid6x4", "dct3": "cube3x4x5", "idct3": "cube3x4x5"}
    port = {"dct1": oracle.port.dct_direct_1d, "idct1": oracle.port.idct_direct_1d,
            "idxst1": oracle.port.idxst_direct_1d, "dct2": oracle.port.dct_2d, "idct2": oracle.port.idct_2d,
            "idct-idxst": oracle.port.idct_idxst_2d, "idxst-idct": oracle.port.idxst_idct_2d,
            "dct3": oracle.port.dct_3d, "idct3": oracle.port.idct_3d}
    for kind, name in cases.items():
        out = tmp_path / f"{kind}.dctb"
        y = dctb.transform_file(os.path.join(FIX, name + ".dctb"), out, kind)
        want = port[kind](EXPECTED[name])
        assert np.array_equal(dctb.read_dctb(out), y)
        assert oracle.rel_l2(y, want) < 1e-12, kind
    for algo in ("4n", "2n-mirrored", "2n-padded"):
        y = dctb.transform_file(os.path.join(FIX, "vec8.dctb"), tmp_path / "v.dctb", "dct1", algo=algo)
        assert oracle.rel_l2(y, oracle.port.dct_direct_1d(EXPECTED["vec8"])) < 1e-12
