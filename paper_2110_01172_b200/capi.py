"""ctypes view of the C ABI (include/sdct_b200.h) — the exact boundary a
reference-side FFI binding would use. Loads the in-tree
paper_2110_01172_b200/lib/libsdct_b200.so and raises if it is missing: there is
no CPU fallback."""
from __future__ import annotations

import ctypes
import os

LIBSO = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libsdct_b200.so")

OK, ERR_SHAPE, ERR_PLAN, ERR_BOUNDS, ERR_CUDA, ERR_OOM, ERR_ARG, ERR_NODEVICE = range(8)
F32, F64 = 0, 1
ORIENT_AUTO, ORIENT_DIRECT, ORIENT_TRANSPOSED = -1, 0, 1
KINDS = {
    "dct_2d": 0, "idct_2d": 1, "idct_idxst_2d": 2, "idxst_idct_2d": 3, "dct_3d": 4,
    "idct_3d": 5, "dct_2d_rowcol": 6, "dct_1d": 7, "idct_1d": 8, "idxst_1d": 9,
    "idct_idxst_2d_rowcol": 10, "idxst_idct_2d_rowcol": 11,
}
RANK_OF = {"dct_2d": 2, "idct_2d": 2, "idct_idxst_2d": 2, "idxst_idct_2d": 2, "dct_2d_rowcol": 2,
           "idct_idxst_2d_rowcol": 2, "idxst_idct_2d_rowcol": 2,
           "dct_3d": 3, "idct_3d": 3, "dct_1d": 1, "idct_1d": 1, "idxst_1d": 1}

# (name, restype, argtypes) for every function declared in include/sdct_b200.h
_VP = ctypes.c_void_p
SIGNATURES = [
    ("sdct_version", ctypes.c_int, []),
    ("sdct_last_error", ctypes.c_char_p, []),
    ("sdct_plan_create", ctypes.c_int, [ctypes.POINTER(_VP), ctypes.c_int, ctypes.POINTER(ctypes.c_int64),
                                        ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int]),
    ("sdct_plan_destroy", ctypes.c_int, [_VP]),
    ("sdct_plan_orientation", ctypes.c_int, [_VP, ctypes.POINTER(ctypes.c_int)]),
    ("sdct_plan_is_fast", ctypes.c_int, [_VP, ctypes.POINTER(ctypes.c_int)]),
    ("sdct_plan_workspace_size", ctypes.c_int, [_VP, ctypes.POINTER(ctypes.c_size_t)]),
    ("sdct_plan_device_bytes", ctypes.c_int, [_VP, ctypes.POINTER(ctypes.c_size_t)]),
    ("sdct_plan_corrupt_twiddle", ctypes.c_int, [_VP, ctypes.c_int64]),
    ("sdct_exec", ctypes.c_int, [_VP, ctypes.c_int, _VP, _VP, _VP, _VP]),
    ("sdct_exec_host", ctypes.c_int, [_VP, ctypes.c_int, _VP, _VP, _VP]),
    ("sdct_force_fields", ctypes.c_int, [_VP, _VP, _VP, _VP, _VP, _VP]),
    ("sdct_force_fields_host", ctypes.c_int, [_VP, _VP, _VP, _VP, _VP]),
    ("sdct_compress", ctypes.c_int, [_VP, _VP, _VP, ctypes.c_double, _VP, _VP, _VP]),
    ("sdct_scratch_size", ctypes.c_int, [_VP, ctypes.POINTER(ctypes.c_size_t)]),
    ("sdct_force_fields_scratch", ctypes.c_int, [_VP, _VP, _VP, _VP, _VP, _VP, _VP]),
    ("sdct_compress_scratch", ctypes.c_int, [_VP, _VP, _VP, ctypes.c_double, _VP, _VP, _VP, _VP]),
    ("sdct_exec_host_pipelined", ctypes.c_int, [_VP, ctypes.POINTER(ctypes.c_int), ctypes.c_int, _VP, ctypes.c_int64,
                                                _VP, ctypes.c_int64, ctypes.c_int64, _VP]),
    ("sdct_transpose", ctypes.c_int, [ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _VP, _VP, _VP]),
    ("sdct_rfft_workspace_size", ctypes.c_int, [_VP, ctypes.POINTER(ctypes.c_size_t)]),
    ("sdct_rfft_nd", ctypes.c_int, [_VP, _VP, _VP, _VP, _VP]),
    ("sdct_irfft_nd", ctypes.c_int, [_VP, _VP, _VP, _VP, _VP]),
    ("sdct_rfft_nd_host", ctypes.c_int, [_VP, _VP, _VP]),
    ("sdct_irfft_nd_host", ctypes.c_int, [_VP, _VP, _VP]),
    ("sdct_dft_naive_host", ctypes.c_int, [ctypes.c_int64, ctypes.c_int, _VP, _VP]),
    ("sdct_stage_count", ctypes.c_int, [_VP, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]),
    ("sdct_exec_stage", ctypes.c_int, [_VP, ctypes.c_int, ctypes.c_int, _VP, _VP, _VP, _VP]),
    ("sdct_counters", ctypes.c_int, [_VP, ctypes.c_int, ctypes.POINTER(ctypes.c_uint64)]),
]

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIBSO):
            raise RuntimeError(f"native library not built: {LIBSO} (run __graft_entry__.build())")
        l = ctypes.CDLL(LIBSO)
        for name, res, args in SIGNATURES:
            fn = getattr(l, name)
            fn.restype = res
            fn.argtypes = args
        _lib = l
    return _lib


class SdctError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def check(rc: int) -> None:
    if rc != OK:
        msg = lib().sdct_last_error().decode()
        if rc in (ERR_SHAPE, ERR_PLAN):
            raise ValueError(msg)
        if rc == ERR_BOUNDS:
            raise IndexError(msg)
        raise SdctError(rc, msg)


class Plan:
    """A C-ABI plan: rank 1..3 item shape, leading batch count, dtype."""

    def __init__(self, dims, batch: int = 1, dtype: int = F64, orientation: int = ORIENT_AUTO,
                 device: int = -1):
        self._h = _VP()
        self.dims = tuple(int(d) for d in dims)
        self.batch = int(batch)
        self.dtype = dtype
        arr = (ctypes.c_int64 * len(self.dims))(*self.dims)
        check(lib().sdct_plan_create(ctypes.byref(self._h), len(self.dims), arr, self.batch, dtype,
                                     orientation, device))

    def close(self):
        if self._h:
            lib().sdct_plan_destroy(self._h)
            self._h = _VP()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    @property
    def fast(self) -> bool:
        v = ctypes.c_int()
        check(lib().sdct_plan_is_fast(self._h, ctypes.byref(v)))
        return bool(v.value)

    @property
    def orientation(self) -> int:
        v = ctypes.c_int()
        check(lib().sdct_plan_orientation(self._h, ctypes.byref(v)))
        return v.value

    @property
    def workspace_bytes(self) -> int:
        v = ctypes.c_size_t()
        check(lib().sdct_plan_workspace_size(self._h, ctypes.byref(v)))
        return v.value

    def stage_count(self, kind: str) -> int:
        v = ctypes.c_int()
        check(lib().sdct_stage_count(self._h, KINDS[kind], ctypes.byref(v)))
        return v.value

    def exec(self, kind: str, d_in: int, d_out: int, workspace: int = 0, stream: int = 0) -> None:
        check(lib().sdct_exec(self._h, KINDS[kind], d_in, d_out, workspace or None, stream or None))

    def exec_stage(self, kind: str, stage: int, d_in: int, d_out: int, workspace: int = 0,
                   stream: int = 0) -> None:
        check(lib().sdct_exec_stage(self._h, KINDS[kind], stage, d_in, d_out, workspace or None,
                                    stream or None))

    def exec_host(self, kind: str, h_in: int, h_out: int, stream: int = 0) -> None:
        check(lib().sdct_exec_host(self._h, KINDS[kind], h_in, h_out, stream or None))

    def corrupt_twiddle(self, index: int) -> None:
        check(lib().sdct_plan_corrupt_twiddle(self._h, index))

    def counters(self, kind: str):
        out = (ctypes.c_uint64 * 5)()
        check(lib().sdct_counters(self._h, KINDS[kind], out))
        return tuple(int(v) for v in out)
