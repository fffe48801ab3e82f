"""TEST INFRASTRUCTURE — the CPU checker for the DCT hot path. NOT PRODUCT CODE.

Two checkers live here, both CPU-only:

* ``port``  — ``oracle/sdct_oracle.c``, a plain-C restatement of the reference
  algorithm (each function cites the reference file:line it follows), built into
  ``oracle/_build/libsdct_oracle.so``.
* ``ref``   — the unmodified reference library compiled from
  ``/root/reference/proj/src`` into ``oracle/_ref/libsdct_ref.so`` by
  ``oracle/Makefile`` (target ``ref``), driven through ``oracle/ref_shim.cpp``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline leg
and ``--impl reference``) may import this package, and only as the checker or
the timed CPU baseline. The product (``paper_2110_01172_b200``) never does.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "libsdct_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsdct_ref.so")
REF_PY = os.path.join(HERE, "_ref", "python")
REFERENCE_SRC = "/root/reference/proj"

# Kind codes shared with oracle/ref_shim.cpp.
KINDS = {
    "dct_2d": 0,
    "idct_2d": 1,
    "idct_idxst_2d": 2,
    "idxst_idct_2d": 3,
    "dct_3d": 4,
    "idct_3d": 5,
    "dct_2d_rowcol": 6,
    "idct_idxst_2d_rowcol": 7,
    "idxst_idct_2d_rowcol": 8,
}


def build(ref: bool | None = None) -> None:
    """Compile the C restatement and (when the reference sources exist) the reference."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)
    if ref is None:
        ref = os.path.isdir(REFERENCE_SRC)
    if ref:
        subprocess.run(["make", "-s", "-j8", "-C", HERE, "ref"], check=True)


_port = None
_ref = None


def _port_lib():
    global _port
    if _port is None:
        if not os.path.exists(PORT_SO):
            build(ref=False)
        lib = ctypes.CDLL(PORT_SO)
        P = ctypes.POINTER(ctypes.c_double)
        S = ctypes.c_size_t
        lib.sdct_oracle_dct_2d.argtypes = [P, S, S, P]
        lib.sdct_oracle_idct_family_2d.argtypes = [P, S, S, ctypes.c_int, P]
        lib.sdct_oracle_dct_3d.argtypes = [P, S, S, S, P]
        lib.sdct_oracle_idct_3d.argtypes = [P, S, S, S, P]
        for name in ("dct_direct_1d", "idct_direct_1d", "idxst_direct_1d"):
            getattr(lib, "sdct_oracle_" + name).argtypes = [P, S, P]
        lib.sdct_oracle_dct_direct_2d.argtypes = [P, S, S, P]
        lib.sdct_oracle_rowcol_2d.argtypes = [P, S, S, ctypes.c_int, P]
        lib.sdct_oracle_force_fields_2d.argtypes = [P, S, S, P, P]
        _port = lib
    return _port


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def _ref_lib():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise RuntimeError(f"reference library not built: {REF_SO} (make -C oracle ref)")
        lib = ctypes.CDLL(REF_SO)
        lib.sdct_ref_run.argtypes = [
            ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_size_t),
            ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
            ctypes.c_uint, ctypes.c_int,
        ]
        lib.sdct_ref_run.restype = ctypes.c_int
        lib.sdct_ref_force.argtypes = [ctypes.c_size_t, ctypes.c_size_t, ctypes.POINTER(ctypes.c_double),
                                       ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                                       ctypes.c_uint, ctypes.c_int]
        lib.sdct_ref_force.restype = ctypes.c_int
        D = ctypes.POINTER(ctypes.c_double)
        lib.sdct_ref_run_timed.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_size_t), D, D,
                                           ctypes.c_uint, ctypes.c_int, D]
        lib.sdct_ref_run_timed.restype = ctypes.c_int
        lib.sdct_ref_force_timed.argtypes = [ctypes.c_size_t, ctypes.c_size_t, D, D, D, ctypes.c_uint,
                                             ctypes.c_int, D]
        lib.sdct_ref_force_timed.restype = ctypes.c_int
        lib.sdct_ref_write_dctb.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(ctypes.c_size_t),
                                            ctypes.POINTER(ctypes.c_double)]
        lib.sdct_ref_write_dctb.restype = ctypes.c_int
        lib.sdct_ref_read_dctb.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_int),
                                           ctypes.POINTER(ctypes.c_size_t), ctypes.POINTER(ctypes.c_double),
                                           ctypes.c_size_t]
        lib.sdct_ref_read_dctb.restype = ctypes.c_int
        lib.sdct_ref_last_error.restype = ctypes.c_char_p
        _ref = lib
    return _ref


def _dp(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _as64(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))


class _Port:
    """C restatement (single-threaded). Leading batch dims are looped over."""

    @staticmethod
    def _batched(x, rank, fn):
        x = _as64(x)
        if x.ndim < rank:
            raise ValueError(f"expected rank >= {rank}")
        lead = x.shape[: x.ndim - rank]
        core = x.shape[x.ndim - rank:]
        xs = x.reshape((-1,) + core)
        out = np.empty_like(xs)
        for b in range(xs.shape[0]):
            xb = np.ascontiguousarray(xs[b])
            yb = np.empty_like(xb)
            fn(xb, core, yb)
            out[b] = yb
        return out.reshape(lead + core)

    def dct_2d(self, x):
        lib = _port_lib()
        return self._batched(x, 2, lambda a, s, o: lib.sdct_oracle_dct_2d(_dp(a), s[0], s[1], _dp(o)))

    def _idct_family(self, x, mode):
        lib = _port_lib()
        return self._batched(
            x, 2, lambda a, s, o: lib.sdct_oracle_idct_family_2d(_dp(a), s[0], s[1], mode, _dp(o)))

    def idct_2d(self, x):
        return self._idct_family(x, 0)

    def idxst_idct_2d(self, x):
        return self._idct_family(x, 1)

    def idct_idxst_2d(self, x):
        return self._idct_family(x, 2)

    def force_demo_fields(self, x):
        """(xi1, xi2) of a rank-2 density (proj/src/force.cpp:11-37)."""
        lib = _port_lib()
        x = _as64(x)
        if x.ndim != 2:
            raise ValueError("force_demo_fields expects a rank-2 density grid")
        xi1, xi2 = np.empty_like(x), np.empty_like(x)
        lib.sdct_oracle_force_fields_2d(_dp(x), x.shape[0], x.shape[1], _dp(xi1), _dp(xi2))
        return xi1, xi2

    def compress(self, x, epsilon: float):
        """Numeric core of compress_image (proj/src/compress.cpp:33-46): zero
        |b| < epsilon of b = dct_2d(x), reconstruct idct_2d(b) * 4/(N1 N2).
        Returns (reconstruction, zeroed count)."""
        b = self.dct_2d(x)
        drop = np.abs(b) < epsilon
        b = np.where(drop, 0.0, b)
        return self.idct_2d(b) * (4.0 / b.size), int(drop.sum())

    def dct_3d(self, x):
        lib = _port_lib()
        return self._batched(
            x, 3, lambda a, s, o: lib.sdct_oracle_dct_3d(_dp(a), s[0], s[1], s[2], _dp(o)))

    def idct_3d(self, x):
        lib = _port_lib()
        return self._batched(
            x, 3, lambda a, s, o: lib.sdct_oracle_idct_3d(_dp(a), s[0], s[1], s[2], _dp(o)))

    def dct_direct_1d(self, x):
        lib = _port_lib()
        return self._batched(x, 1, lambda a, s, o: lib.sdct_oracle_dct_direct_1d(_dp(a), s[0], _dp(o)))

    def idct_direct_1d(self, x):
        lib = _port_lib()
        return self._batched(x, 1, lambda a, s, o: lib.sdct_oracle_idct_direct_1d(_dp(a), s[0], _dp(o)))

    def idxst_direct_1d(self, x):
        lib = _port_lib()
        return self._batched(x, 1, lambda a, s, o: lib.sdct_oracle_idxst_direct_1d(_dp(a), s[0], _dp(o)))

    def _rowcol(self, x, kind):
        lib = _port_lib()
        return self._batched(x, 2, lambda a, s, o: lib.sdct_oracle_rowcol_2d(_dp(a), s[0], s[1], kind, _dp(o)))

    def dct_2d_rowcol(self, x):
        """dct_rows + transpose twice (proj/src/dct2d.cpp:395-406)."""
        return self._rowcol(x, 0)

    def idct_idxst_2d_rowcol(self, x):
        """composite_2d_rowcol, IdctIdxst (proj/src/transforms_ext.cpp:287-301)."""
        return self._rowcol(x, 1)

    def idxst_idct_2d_rowcol(self, x):
        """composite_2d_rowcol, IdxstIdct (proj/src/transforms_ext.cpp:287-301)."""
        return self._rowcol(x, 2)

    def dct_direct_2d(self, x):
        lib = _port_lib()
        return self._batched(x, 2, lambda a, s, o: lib.sdct_oracle_dct_direct_2d(_dp(a), s[0], s[1], _dp(o)))


class _Ref:
    """The unmodified reference (oracle/_ref/libsdct_ref.so), prebuilt plans.

    ``threads=0`` means the reference's own default (all hardware threads,
    proj/src/exec.cpp:8-12)."""

    def run(self, kind: str, x, threads: int = 0, reps: int = 1) -> np.ndarray:
        lib = _ref_lib()
        x = _as64(x)
        dims = (ctypes.c_size_t * x.ndim)(*x.shape)
        out = np.empty_like(x)
        rc = lib.sdct_ref_run(KINDS[kind], x.ndim, dims, _dp(x), _dp(out), threads, reps)
        if rc != 0:
            msg = lib.sdct_ref_last_error().decode()
            raise ValueError(msg) if rc == 1 else RuntimeError(msg)
        return out

    def run_timed(self, kind: str, x, threads: int = 0, reps: int = 1):
        """(output, seconds per call): plan and input tensor built once outside
        the clock, `reps` calls of the transform timed inside the reference."""
        lib = _ref_lib()
        x = _as64(x)
        dims = (ctypes.c_size_t * x.ndim)(*x.shape)
        out = np.empty_like(x)
        sec = ctypes.c_double(0.0)
        rc = lib.sdct_ref_run_timed(KINDS[kind], x.ndim, dims, _dp(x), _dp(out), threads, reps, ctypes.byref(sec))
        if rc != 0:
            msg = lib.sdct_ref_last_error().decode()
            raise ValueError(msg) if rc == 1 else RuntimeError(msg)
        return out, sec.value / reps

    def force_timed(self, x, threads: int = 0, reps: int = 1):
        """((xi1, xi2), seconds per call) of force_demo_fields, input built once."""
        lib = _ref_lib()
        x = _as64(x)
        xi1, xi2 = np.empty_like(x), np.empty_like(x)
        sec = ctypes.c_double(0.0)
        rc = lib.sdct_ref_force_timed(x.shape[0], x.shape[1], _dp(x), _dp(xi1), _dp(xi2), threads, reps,
                                      ctypes.byref(sec))
        if rc != 0:
            raise RuntimeError(lib.sdct_ref_last_error().decode())
        return (xi1, xi2), sec.value / reps

    def force_demo_fields(self, x, threads: int = 0, reps: int = 1):
        lib = _ref_lib()
        x = _as64(x)
        if x.ndim != 2:
            raise ValueError("force_demo_fields expects a rank-2 density grid")
        xi1, xi2 = np.empty_like(x), np.empty_like(x)
        rc = lib.sdct_ref_force(x.shape[0], x.shape[1], _dp(x), _dp(xi1), _dp(xi2), threads, reps)
        if rc != 0:
            msg = lib.sdct_ref_last_error().decode()
            raise ValueError(msg) if rc == 1 else RuntimeError(msg)
        return xi1, xi2

    def write_dctb(self, path: str, x) -> int:
        """sdct::write_dctb (proj/src/io.cpp:96-107); returns the shim status
        (0 ok, 1 ShapeError, 3 FormatError)."""
        lib = _ref_lib()
        x = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
        dims = (ctypes.c_size_t * max(x.ndim, 1))(*x.shape)
        return lib.sdct_ref_write_dctb(os.fsencode(path), x.ndim, dims, _dp(x))

    def read_dctb(self, path: str):
        """sdct::read_dctb (proj/src/io.cpp:60-94): (status, array or None);
        status 0 ok, 3 FormatError."""
        lib = _ref_lib()
        rank = ctypes.c_int(0)
        dims = (ctypes.c_size_t * 4)()
        rc = lib.sdct_ref_read_dctb(os.fsencode(path), ctypes.byref(rank), dims, None, 0)
        if rc != 0:
            return rc, None
        out = np.empty(tuple(dims[: rank.value]), dtype=np.float64)
        rc = lib.sdct_ref_read_dctb(os.fsencode(path), ctypes.byref(rank), dims, _dp(out), out.size)
        return rc, out

    def __getattr__(self, name):
        if name in KINDS:
            return lambda x, threads=0: self.run(name, x, threads)
        raise AttributeError(name)


port = _Port()
ref = _Ref()


def rel_l2(got, want) -> float:
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    den = float(np.linalg.norm(want.ravel()))
    num = float(np.linalg.norm((got - want).ravel()))
    return num / den if den > 0 else num


def max_rel(got, want) -> float:
    """The reference's own metric: max|got-want| / max|want| (test_dct2d.cpp:25-33)."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    err = float(np.max(np.abs(got - want))) if got.size else 0.0
    scale = float(np.max(np.abs(want))) if want.size else 0.0
    return err / scale if scale > 1e-12 else err
