"""CPU tests of the boundary and host logic: the C-ABI library loads and
exports every symbol include/sdct_b200.h declares, argument validation happens
before any device work, the python package refuses to run without a GPU (no
CPU fallback), and the shared-memory swizzles are conflict free."""
import os
import re

import numpy as np
import pytest

from tests import swizzle_model as sm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "sdct_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sdct_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    import ctypes

    from paper_2110_01172_b200 import capi

    lib = ctypes.CDLL(capi.LIBSO)
    syms = _declared_symbols()
    assert len(syms) >= 13
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in include/sdct_b200.h but not exported"
    # the ctypes binding covers exactly the declared surface
    assert sorted(n for n, _, _ in capi.SIGNATURES) == syms


def test_version_and_error_channel():
    from paper_2110_01172_b200 import capi

    assert capi.lib().sdct_version() >= 10000
    assert isinstance(capi.lib().sdct_last_error(), bytes)


def test_plan_validation_precedes_device_checks():
    from paper_2110_01172_b200 import capi

    with pytest.raises(ValueError, match="positive"):
        capi.Plan((0, 4))
    with pytest.raises(ValueError, match="rank"):
        capi.Plan((2, 2, 2, 2))
    with pytest.raises(ValueError, match="batch"):
        capi.Plan((4, 4), batch=0)


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible; this checks the CPU-only container")
    import paper_2110_01172_b200 as sd
    from paper_2110_01172_b200 import capi

    with pytest.raises(capi.SdctError) as ei:
        capi.Plan((8, 8))
    assert ei.value.code == capi.ERR_NODEVICE
    with pytest.raises(sd.DeviceError):
        sd.dct_2d(np.zeros((8, 8)))


def test_reference_error_types():
    import paper_2110_01172_b200 as sd

    assert issubclass(sd.ShapeError, ValueError)
    assert issubclass(sd.FormatError, ValueError)
    with pytest.raises(ValueError):
        sd.dct_2d(np.zeros(8))  # rank error is raised before any device work
    with pytest.raises(ValueError):
        sd.dct_1d(np.zeros((2, 2, 2, 2, 2)))
    with pytest.raises(ValueError):
        sd.amdahl_speedup(1.5, 2.0)
    assert sd.amdahl_speedup(0.5, 2.0) == pytest.approx(4 / 3)


def test_reference_python_surface_names():
    import paper_2110_01172_b200 as sd

    # the reference module's 17 exports (proj/python/sdct/__init__.py:8-26)
    for name in ["ShapeError", "FormatError", "amdahl_speedup", "dct_1d", "dct_2d", "dct_2d_rowcol",
                 "dct_3d", "dct_4d", "dct_oracle_1d", "dct_oracle_2d", "force_demo_fields", "idct_1d",
                 "idct_2d", "idct_3d", "idct_idxst_2d", "idxst_1d", "idxst_idct_2d"]:
        assert hasattr(sd, name), name


@pytest.mark.parametrize("esize", [8, 16])
def test_swizzle_conflict_free(esize):
    # every DIF stage of every tile geometry the plans pick (pick_lgw in plan.cu)
    for L in (16, 64, 256, 1024, 2048, 4096):
        for nl in (2, 4, 8, 16, 32):
            if L * nl * esize > 128 * 1024:
                continue
            assert sm.stage_degrees(L, nl, 256, esize, True) == [1] * sm.radix_plan(L)[0], (L, nl)
        for g in (2, 4):
            assert sm.stage_degrees(L, g, 256, esize, False) == [1] * sm.radix_plan(L)[0], (L, g)


def test_swizzle_is_a_bijection():
    for esize in (8, 16):
        for n in (1 << 10, 1 << 13):
            for f in (sm.swz_col, sm.swz_row):
                assert sorted(f(a, esize) for a in range(n)) == list(range(n))


def test_digit_reversal_is_a_permutation():
    for L in (2, 8, 32, 512, 2048, 4096):
        assert sorted(sm.digit_pos(L, k) for k in range(L)) == list(range(L))


def test_cpp_api_program_is_built():
    # the C++ drop-in check links against the library without a GPU present
    import os

    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                       "paper_2110_01172_b200", "lib", "api_smoke")
    assert os.path.exists(exe)


def test_fastdiv_formula():
    # kernels_generic.cu FastDiv: q = (umulhi(x, m) + x) >> s with
    # s = ceil(log2 d), m = floor(2^32 (2^s - d) / d) + 1, for 0 <= x < 2^31
    rng = np.random.default_rng(5)
    ds = list(range(1, 70)) + [125, 250, 1000, 2000, 2047, 2049, 4093, 4095, 4096, 4097, 65535, 1 << 20,
                                (1 << 31) - 1] + rng.integers(1, 1 << 31, 200).tolist()
    for d in ds:
        s = 0
        while (1 << s) < d:
            s += 1
        m = ((1 << 32) * ((1 << s) - d)) // d + 1
        assert m < (1 << 32)
        ks = np.unique(np.concatenate([np.arange(0, 4), rng.integers(0, ((1 << 31) - 2) // d + 1, 40)]))
        edges = np.concatenate([ks * d - 1, ks * d, ks * d + 1])  # around multiples of d
        edges = edges[(edges >= 0) & (edges < (1 << 31))]
        xs = np.concatenate([rng.integers(0, 1 << 31, 300), edges, np.array([(1 << 31) - 1, (1 << 31) - 2])])
        for x in xs.tolist():
            q = ((((x * m) >> 32) + x) & 0xFFFFFFFF) >> s
            assert q == x // d, (d, x)


def _rowp_k0(t: int, M: int) -> int:
    # mirror of rowp_k0 (paper_2110_01172_b200/csrc/kernels_rowp.cuh)
    K0, w, l = M // 8, t >> 5, t & 31
    if l < 16:
        return 16 * w + l
    u = 16 * w + l - 16
    return K0 // 2 if u == 0 else K0 - u


@pytest.mark.parametrize("M", [1024, 2048])
def test_rowp_mirror_pairing_and_banks(M):
    # mirror-paired row kernel: every k0 once, lane ^ 16 holds the mirror set
    # (k0 + k0' = M/8, or both self-mirrors), and the paired radix-8 stage's
    # shared-memory accesses are at most 2-way conflicted (fp64 row swizzle)
    K0 = NT = M // 8
    ks = [_rowp_k0(t, M) for t in range(NT)]
    assert sorted(ks) == list(range(K0))
    for t in range(NT):
        a, b = ks[t], ks[t ^ 16]
        assert (a + b) % K0 == 0 or {a, b} <= {0, K0 // 2}
    for line in (0, 1):
        for t0 in range(0, NT, 32):
            for r in range(8):
                addrs = [sm.row_at(line, 8 * (sm.digit_pos(M, ks[t]) >> 3) + r, M, 16) for t in range(t0, t0 + 32)]
                assert sm.conflict_degree(addrs, 16) <= 2
