"""CPU tests of the checker itself: the C restatement (oracle/sdct_oracle.c)
pinned against golden vectors produced by the unmodified reference
(tests/golden/make_golden.py), against scipy.fft, against the reference's
known answers, and against the brute-force direct sums. No GPU involved."""
import numpy as np
import pytest
import scipy.fft as sf

import oracle

KINDS_2D = ["dct_2d", "idct_2d", "idct_idxst_2d", "idxst_idct_2d"]


def _keys(golden, prefix):
    return sorted(k.split("/", 1)[1] for k in golden if k.startswith(prefix + "/"))


@pytest.mark.parametrize("kind", KINDS_2D)
def test_port_matches_reference_golden_2d(golden, kind):
    keys = _keys(golden, kind)
    assert len(keys) >= 80
    for key in keys:
        x = golden["in/" + key]
        got = getattr(oracle.port, kind)(x)
        want = golden[f"{kind}/{key}"]
        # Direct-orientation shapes are bit-identical to the reference; the
        # reference auto-transposes row-dominant shapes (dct2d.cpp:294-298),
        # which only reorders rounding.
        assert oracle.max_rel(got, want) < 1e-13, (kind, key)


def test_port_matches_rowcol_golden(golden):
    for key in _keys(golden, "dct_2d_rowcol"):
        x = golden["in/" + key]
        assert oracle.max_rel(oracle.port.dct_2d(x), golden["dct_2d_rowcol/" + key]) < 1e-12, key


@pytest.mark.parametrize("kind", ["dct_3d", "idct_3d"])
def test_port_matches_reference_golden_3d(golden, kind):
    keys = _keys(golden, kind)
    assert len(keys) >= 10
    for key in keys:
        x = golden["in/" + key]
        assert oracle.max_rel(getattr(oracle.port, kind)(x), golden[f"{kind}/{key}"]) < 1e-13, key


def test_direct_orientation_is_bit_exact(golden):
    # square / column-dominant shapes run Direct in the reference -> identical bits
    for key in ("8x8", "7x5", "64x64", "31x17", "33x17", "128x128", "64x256"):
        x = golden["in/" + key]
        assert np.array_equal(oracle.port.dct_2d(x), golden["dct_2d/" + key]), key
        assert np.array_equal(oracle.port.idct_2d(x), golden["idct_2d/" + key]), key


def test_known_answers(golden):
    # SPEC.md:418-419, proj/tests/cli_tests.sh:113-121
    np.testing.assert_allclose(oracle.port.dct_2d(np.ones((2, 2))), [[4, 0], [0, 0]], atol=1e-15)
    d = np.zeros((2, 2))
    d[0, 0] = 1
    s = np.sqrt(2) / 2
    np.testing.assert_allclose(oracle.port.dct_2d(d), [[1, s], [s, 0.5]], atol=1e-15)
    # proj/tests/test_transforms_ext.cpp:180-185
    y = oracle.port.dct_3d(np.ones((2, 2, 2)))
    assert abs(y[0, 0, 0] - 8) < 1e-12 and np.abs(y.ravel()[1:]).max() < 1e-12
    np.testing.assert_allclose(golden["kat/ones2x2/dct_2d"], [[4, 0], [0, 0]], atol=1e-15)


@pytest.mark.parametrize("shape", [(24, 17), (64, 64), (9, 14), (1, 5), (5, 1)])
def test_scipy_identities_2d(shape):
    x = np.random.default_rng(20240815).uniform(-1, 1, shape)
    np.testing.assert_allclose(oracle.port.dct_2d(x), sf.dctn(x, type=2) / 4, atol=1e-12)
    np.testing.assert_allclose(oracle.port.idct_2d(x), sf.dctn(x, type=3) / 4, atol=1e-12)


def test_scipy_identity_3d():
    x = np.random.default_rng(5).uniform(-1, 1, (5, 6, 7))
    np.testing.assert_allclose(oracle.port.dct_3d(x), sf.dctn(x, type=2) / 8, atol=1e-12)


def test_round_trips():
    rng = np.random.default_rng(3)
    for shape in [(1, 1), (2, 2), (9, 14), (8, 8), (16, 3)]:
        x = rng.uniform(-1, 1, shape)
        back = oracle.port.idct_2d(oracle.port.dct_2d(x))
        np.testing.assert_allclose(back, x * shape[0] * shape[1] / 4, atol=1e-10)
    for shape in [(2, 3, 4), (5, 4, 3), (8, 8, 8)]:
        x = rng.uniform(-1, 1, shape)
        back = oracle.port.idct_3d(oracle.port.dct_3d(x))
        np.testing.assert_allclose(back, x * np.prod(shape) / 8, atol=1e-10)


def test_direct_sum_oracles():
    rng = np.random.default_rng(9)
    for shape in [(1, 1), (3, 5), (8, 8), (16, 12)]:
        x = rng.uniform(-1, 1, shape)
        assert oracle.max_rel(oracle.port.dct_2d(x), oracle.port.dct_direct_2d(x)) < 1e-10


def test_composites_separable():
    # proj/tests/test_transforms_ext.cpp:126-134: composites == separable 1D oracles
    x = np.random.default_rng(80).uniform(-1, 1, (6, 5))
    idct0 = np.stack([oracle.port.idct_direct_1d(np.ascontiguousarray(c)) for c in x.T]).T
    want_ci = np.stack([oracle.port.idxst_direct_1d(r) for r in idct0])
    assert oracle.max_rel(oracle.port.idct_idxst_2d(x), want_ci) < 1e-10
    idxst0 = np.stack([oracle.port.idxst_direct_1d(np.ascontiguousarray(c)) for c in x.T]).T
    want_ic = np.stack([oracle.port.idct_direct_1d(r) for r in idxst0])
    assert oracle.max_rel(oracle.port.idxst_idct_2d(x), want_ic) < 1e-10


def test_idxst_definition():
    n = 12
    x = np.random.default_rng(1).uniform(-1, 1, n)
    k = np.arange(n)[:, None]
    m = np.arange(1, n)[None, :]
    want = (x[1:][None, :] * np.sin(np.pi / n * m * (k + 0.5))).sum(axis=1)
    np.testing.assert_allclose(oracle.port.idxst_direct_1d(x), want, atol=1e-12)


def test_reference_library_agrees_when_built():
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built (make -C oracle ref)")
    x = np.random.default_rng(2).uniform(-1, 1, (64, 48))
    for kind in KINDS_2D:
        assert np.array_equal(getattr(oracle.port, kind)(x), oracle.ref.run(kind, x)), kind


@pytest.mark.parametrize("shape", [(1, 1), (1, 5), (3, 1), (2, 8), (7, 9), (8, 8), (16, 12), (31, 17), (64, 48)])
def test_port_rowcol_bitwise_equals_reference(shape):
    # dct_rows / inverse_rows + transposes (dct2d.cpp:248-290,395-406,
    # transforms_ext.cpp:40-88,287-311) restated in C vs the unmodified reference
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built (make -C oracle ref)")
    x = np.random.default_rng(7).uniform(-1, 1, shape)
    for kind, fused in (("dct_2d_rowcol", "dct_2d"), ("idct_idxst_2d_rowcol", "idct_idxst_2d"),
                        ("idxst_idct_2d_rowcol", "idxst_idct_2d")):
        got = getattr(oracle.port, kind)(x)
        assert np.array_equal(got, oracle.ref.run(kind, x)), (kind, shape)
        # and the row-column forms agree with the fused ones (acceptance.cpp:291-321)
        assert oracle.max_rel(got, getattr(oracle.port, fused)(x)) <= 1e-10, (kind, shape)


def test_port_force_fields_match_reference_golden(golden):
    # proj/src/force.cpp:11-37 through the reference's pybind module
    keys = _keys(golden, "force_xi1")
    assert len(keys) > 60
    for key in keys:
        xi1, xi2 = oracle.port.force_demo_fields(golden["in/" + key])
        assert oracle.rel_l2(xi1, golden["force_xi1/" + key]) <= 1e-13, key
        assert oracle.rel_l2(xi2, golden["force_xi2/" + key]) <= 1e-13, key


def test_port_compress_matches_reference_composition():
    # compress.cpp:33-46 restated: reference dct_2d, threshold, reference
    # idct_2d, 4/(N1 N2) — against the port's own composition
    if not oracle.ref_available():
        pytest.skip("reference library not built")
    x = np.random.default_rng(5).uniform(-1, 1, (24, 17))
    b = oracle.ref.run("dct_2d", x)
    eps = float(np.median(np.abs(b)))
    want = oracle.ref.run("idct_2d", np.where(np.abs(b) < eps, 0.0, b)) * (4.0 / x.size)
    got, zeroed = oracle.port.compress(x, eps)
    assert oracle.rel_l2(got, want) <= 1e-13
    assert zeroed == int((np.abs(b) < eps).sum())
    r0, z0 = oracle.port.compress(x, 0.0)
    assert z0 == 0 and oracle.rel_l2(r0, x) <= 1e-13
