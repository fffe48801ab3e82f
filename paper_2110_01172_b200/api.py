"""Dispatch between the reference-compatible numpy surface (``_sdct``) and the
device path for torch CUDA tensors (cached ``_sdct.Plan`` per shape/dtype/device,
workspace from torch's caching allocator on the current stream)."""
from __future__ import annotations

import os
import threading
from collections import OrderedDict

from . import _sdct

_KIND = {
    "dct_1d": _sdct.DCT_1D, "idct_1d": _sdct.IDCT_1D, "idxst_1d": _sdct.IDXST_1D,
    "dct_2d": _sdct.DCT_2D, "idct_2d": _sdct.IDCT_2D, "idct_idxst_2d": _sdct.IDCT_IDXST_2D,
    "idxst_idct_2d": _sdct.IDXST_IDCT_2D, "dct_2d_rowcol": _sdct.DCT_2D_ROWCOL,
    "idct_idxst_2d_rowcol": _sdct.IDCT_IDXST_2D_ROWCOL, "idxst_idct_2d_rowcol": _sdct.IDXST_IDCT_2D_ROWCOL,
    "dct_3d": _sdct.DCT_3D, "idct_3d": _sdct.IDCT_3D,
    "dct_axis0": _sdct.DCT_AXIS0, "idct_axis0": _sdct.IDCT_AXIS0,
}
_RANK = {"dct_1d": 1, "idct_1d": 1, "idxst_1d": 1, "dct_3d": 3, "idct_3d": 3}

_plans: "OrderedDict" = OrderedDict()
_lock = threading.Lock()
PLAN_CACHE_MAX = 32
PLAN_CACHE_BYTES = int(os.environ.get("SDCT_PLAN_CACHE_BYTES", str(2 << 30)))


def plan_for(dims, batch: int = 1, dtype: str = "float64", device: int = 0):
    """Cached device plan for ``batch`` items of shape ``dims`` (LRU; bounded
    by PLAN_CACHE_MAX entries and PLAN_CACHE_BYTES of device memory the cached
    plans own — tables plus whatever they allocated on first use)."""
    key = (tuple(int(d) for d in dims), int(batch), dtype, int(device))
    with _lock:
        p = _plans.get(key)
        if p is not None:  # hit: no per-call walk over the cache
            _plans.move_to_end(key)
            return p
        import torch

        with torch.cuda.device(device):
            p = _sdct.Plan(list(key[0]), key[1], dtype)
        _plans[key] = p
        # bounds checked on insertion (plans grow lazily after their first use,
        # so the byte total is re-read from every cached plan here)
        total = sum(q.device_bytes for q in _plans.values())
        while len(_plans) > 1 and (len(_plans) > PLAN_CACHE_MAX or total > PLAN_CACHE_BYTES):
            _, old = _plans.popitem(last=False)
            total -= old.device_bytes
        return p


def _is_torch_cuda(x) -> bool:
    t = type(x)
    return t.__module__.startswith("torch") and getattr(x, "is_cuda", False)


def _device_call(name: str, x):
    import torch

    rank = _RANK.get(name, 2)
    if x.dim() < rank:
        raise ShapeError(f"{name} expects a rank-{rank} tensor (plus optional batch dims), got {tuple(x.shape)}")
    if x.dtype not in (torch.float32, torch.float64):
        raise ValueError(f"{name}: dtype must be float32 or float64, got {x.dtype}")
    x = x.contiguous()
    if x.data_ptr() % 16:
        x = x.clone()  # the kernels move rows with 16-B bulk copies / TMA
    core = tuple(x.shape[x.dim() - rank:])
    batch = 1
    for d in x.shape[: x.dim() - rank]:
        batch *= int(d)
    if batch == 0 or any(d == 0 for d in core):
        raise ShapeError("tensor extents must be positive")
    dt = "float32" if x.dtype == torch.float32 else "float64"
    dev = x.device.index if x.device.index is not None else torch.cuda.current_device()
    plan = plan_for(core, batch, dt, dev)
    out = torch.empty_like(x)
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev)
        ws = torch.empty(plan.workspace_bytes, dtype=torch.uint8, device=x.device)
        plan.run(_KIND[name], x.data_ptr(), out.data_ptr(), stream.cuda_stream, ws.data_ptr())
    return out


ShapeError = _sdct.ShapeError


def dct_axis0(x):
    """The reference's N-point ``dct_1d`` (proj/src/dct1d.cpp) applied to every
    column of a rank-2 torch CUDA tensor (n1 x m, optional leading batch dims;
    n1 a power of two in [8, 4096], m a multiple of 32 bytes' worth of
    elements): one persistent column pass (kernels_col1d.cuh). The axis-0 leg
    of the slab-decomposed 3D transform (slab3d.py)."""
    if not _is_torch_cuda(x):
        raise TypeError("dct_axis0 takes a torch CUDA tensor")
    return _device_call("dct_axis0", x) if _axis0_ok(x) else _axis0_by_transpose(dct_1d, x)


def idct_axis0(x):
    """The reference's ``idct_1d`` (idct_1d(dct_1d(x)) == n1/2 x) along axis 0
    of every column; same shapes as :func:`dct_axis0`."""
    if not _is_torch_cuda(x):
        raise TypeError("idct_axis0 takes a torch CUDA tensor")
    return _device_call("idct_axis0", x) if _axis0_ok(x) else _axis0_by_transpose(idct_1d, x)


def _axis0_ok(x) -> bool:
    """Shapes the axis-0 column pass takes (else: transpose, contiguous 1D
    transform on the generic GPU path, transpose back)."""
    if x.dim() < 2:
        raise ShapeError(f"axis-0 transforms expect a rank-2 tensor (plus optional batch dims), got {tuple(x.shape)}")
    n1, m = int(x.shape[-2]), int(x.shape[-1])
    return 8 <= n1 <= 4096 and (n1 & (n1 - 1)) == 0 and (m * x.element_size()) % 32 == 0


def _axis0_by_transpose(f, x):
    return f(x.transpose(-1, -2).contiguous()).transpose(-1, -2).contiguous()


def _make(name: str, with_variant: bool = False):
    host = getattr(_sdct, name)

    if with_variant:
        def fn(x, variant: str = "n", threads: int = 0):
            if _is_torch_cuda(x):
                return _device_call(name, x)
            return host(x, variant=variant, threads=threads)
    else:
        def fn(x, threads: int = 0):
            if _is_torch_cuda(x):
                return _device_call(name, x)
            return host(x, threads=threads)

    fn.__name__ = name
    fn.__qualname__ = name
    fn.__doc__ = host.__doc__
    return fn


dct_1d = _make("dct_1d", with_variant=True)
idct_1d = _make("idct_1d")
idxst_1d = _make("idxst_1d")
dct_2d = _make("dct_2d")
dct_2d_rowcol = _make("dct_2d_rowcol")
idct_idxst_2d_rowcol = _make("idct_idxst_2d_rowcol")
idxst_idct_2d_rowcol = _make("idxst_idct_2d_rowcol")
idct_2d = _make("idct_2d")
idct_idxst_2d = _make("idct_idxst_2d")
idxst_idct_2d = _make("idxst_idct_2d")
dct_3d = _make("dct_3d")
idct_3d = _make("idct_3d")


def stream_host(kinds, x, out=None, count=None, device: int = 0, sync: bool = True):
    """Host-resident items through a chain of transforms on the GPU, with the
    copies overlapped: item i+1's host->device copy, item i's kernels and item
    i-1's device->host copy run concurrently (sdct_exec_host_pipelined).

    kinds: transform names applied in order, e.g. ["dct_2d", "idct_2d"].
    x:     CPU torch tensor (pin_memory() for overlap) of shape (items, *dims);
           a leading extent of 1 with count > 1 re-sends the same item.
    out:   CPU tensor for the results (same item shape); allocated pinned if
           None; a leading extent of 1 keeps only the last result.
    sync:  wait for completion (False: stream-ordered on the current stream).
    """
    import torch

    names = [kinds] if isinstance(kinds, str) else list(kinds)
    rank = _RANK.get(names[0], 2)
    if any(_RANK.get(n, 2) != rank for n in names):
        raise ShapeError("stream_host: every transform in the chain must have the same rank")
    if x.is_cuda or x.dim() != rank + 1:
        raise ShapeError(f"stream_host expects a CPU tensor of shape (items, *dims) with {rank} dims per item")
    if x.dtype not in (torch.float32, torch.float64):
        raise ValueError(f"stream_host: dtype must be float32 or float64, got {x.dtype}")
    x = x.contiguous()
    n = int(count) if count is not None else int(x.shape[0])
    if out is None:
        out = torch.empty((1 if x.shape[0] == 1 and n > 1 else n, *x.shape[1:]), dtype=x.dtype).pin_memory()
    if out.dtype != x.dtype or tuple(out.shape[1:]) != tuple(x.shape[1:]) or not out.is_contiguous():
        raise ShapeError("stream_host: out must be a contiguous tensor with the input's item shape and dtype")
    if (x.shape[0] not in (1, n)) or (out.shape[0] not in (1, n)):
        raise ShapeError("stream_host: leading extents must be 1 or the item count")
    item = x[0].numel() * x.element_size()
    dt = "float32" if x.dtype == torch.float32 else "float64"
    plan = plan_for(tuple(x.shape[1:]), 1, dt, device)
    with torch.cuda.device(device):
        stream = torch.cuda.current_stream(device)
        plan.run_host_pipelined([_KIND[k] for k in names], x.data_ptr(), 0 if x.shape[0] == 1 else item,
                                out.data_ptr(), 0 if out.shape[0] == 1 else item, n, stream.cuda_stream)
        if sync:
            stream.synchronize()
    return out


def force_demo_fields(density, threads: int = 0):
    """DREAMPlace-style spectral force fields (xi1, xi2) of a rank-2 density
    (proj/src/force.cpp:11-37): numpy in -> numpy tuple (host copies); a torch
    CUDA tensor (fp32/fp64, optional leading batch dims) -> tensors on the same
    device and stream, with the field weighting fused into the inverse passes."""
    if not _is_torch_cuda(density):
        return _sdct.force_demo_fields(density, threads=threads)
    import torch

    x = density
    if x.dim() < 2:
        raise ShapeError(f"force_demo_fields expects a rank-2 tensor (plus optional batch dims), got {tuple(x.shape)}")
    if x.dtype not in (torch.float32, torch.float64):
        raise ValueError(f"force_demo_fields: dtype must be float32 or float64, got {x.dtype}")
    x = x.contiguous()
    if x.data_ptr() % 16:
        x = x.clone()
    core = tuple(x.shape[-2:])
    batch = 1
    for d in x.shape[:-2]:
        batch *= int(d)
    dt = "float32" if x.dtype == torch.float32 else "float64"
    dev = x.device.index if x.device.index is not None else torch.cuda.current_device()
    plan = plan_for(core, batch, dt, dev)
    xi1, xi2 = torch.empty_like(x), torch.empty_like(x)
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev)
        ws = torch.empty(plan.workspace_bytes, dtype=torch.uint8, device=x.device)
        # per-call coefficient scratch from the caching allocator: concurrent
        # calls on the shared cached plan from other streams stay independent
        scratch = torch.empty(plan.scratch_bytes, dtype=torch.uint8, device=x.device)
        plan.force_fields(x.data_ptr(), xi1.data_ptr(), xi2.data_ptr(), stream.cuda_stream, ws.data_ptr(),
                          scratch.data_ptr())
    return xi1, xi2


# ---- remaining names of the reference module (proj/python/sdct/__init__.py) --
def _to_device(x):
    """(tensor on the GPU, was_numpy) for numpy or torch input (float64 for numpy)."""
    import numpy as np
    import torch

    if _is_torch_cuda(x):
        return x, False
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    return torch.from_numpy(a).to("cuda"), True


def dct_4d(x, threads: int = 0):
    """Rank-4 DCT as two rounds of fused 2D transforms over the axis pairs
    (0, 1) and (2, 3) (proj/src/transforms_ext.cpp:396-425, module.cpp:144-149):
    both rounds are one batched dct_2d launch each; the axis-pair regrouping is
    a device transpose."""
    t, was_np = _to_device(x)
    if t.dim() != 4:
        raise ShapeError(f"dct_nd_factorized expects a rank-4 tensor, got shape {tuple(t.shape)}")
    d0, d1, d2, d3 = (int(s) for s in t.shape)
    # round one, axes (0, 1): [d0 d1][d2 d3] -> [d2 d3][d0][d1], transform, back
    r1 = _device_call("dct_2d", t.reshape(d0 * d1, d2 * d3).t().contiguous().reshape(d2 * d3, d0, d1))
    r1 = r1.reshape(d2 * d3, d0 * d1).t().contiguous().reshape(d0 * d1, d2, d3)
    # round two, axes (2, 3): contiguous inner matrices
    y = _device_call("dct_2d", r1).reshape(d0, d1, d2, d3)
    return y.cpu().numpy() if was_np else y


def _cos_matrix(n: int, device, inverse: bool = False):
    import math

    import torch

    k = torch.arange(n, dtype=torch.float64, device=device)
    if not inverse:  # C[k, n] = cos(pi/N (n + 1/2) k)
        return torch.cos(math.pi / n * torch.outer(k, k + 0.5))
    raise ValueError("only the forward cosine matrix is used")


def dct_oracle_1d(x):
    """Direct quadratic cosine-sum reference y(k) = sum_n x(n) cos(pi/N (n+1/2) k)
    (proj/include/sdct/oracle.hpp:22-24), evaluated on the GPU as one dense
    product with the cosine matrix (no FFT involved)."""
    t, was_np = _to_device(x)
    if t.dim() != 1 or t.numel() == 0:
        raise ShapeError(f"dct_oracle_1d expects a non-empty rank-1 array, got shape {tuple(t.shape)}")
    y = _cos_matrix(t.numel(), t.device) @ t.double()
    return y.cpu().numpy() if was_np else y.to(t.dtype)


def dct_oracle_2d(x):
    """Direct quadruple-sum reference y(k1,k2) = sum_{n1,n2} x(n1,n2)
    cos(pi/N1 (n1+1/2) k1) cos(pi/N2 (n2+1/2) k2) (oracle.hpp:30-32), evaluated
    as C1 x C2^T on the GPU."""
    t, was_np = _to_device(x)
    if t.dim() != 2 or t.numel() == 0:
        raise ShapeError(f"dct_oracle_2d expects a non-empty rank-2 array, got shape {tuple(t.shape)}")
    y = _cos_matrix(t.shape[0], t.device) @ t.double() @ _cos_matrix(t.shape[1], t.device).t()
    return y.cpu().numpy() if was_np else y.to(t.dtype)


def compress(x, epsilon: float):
    """Frequency-domain compression of a rank-2 array (the numeric core of
    proj/src/compress.cpp:24-54): zero every 2D DCT coefficient with
    |b| < epsilon, reconstruct with idct_2d * 4/(N1 N2). Returns
    (reconstruction, stats) with stats = {total_coefficients,
    zeroed_coefficients, zeroed_fraction}. The threshold and normalisation are
    fused into the inverse row kernels (sdct_compress); 8-bit rounding, PSNR
    and the PGM I/O of the reference's image app are not part of this path."""
    import math

    import torch

    t, was_np = _to_device(x)
    if t.dim() != 2:
        raise ShapeError(f"compress expects a rank-2 array, got shape {tuple(t.shape)}")
    if math.isnan(epsilon) or epsilon < 0:
        raise ValueError("compress: epsilon must be >= 0")
    if t.dtype not in (torch.float32, torch.float64):
        raise ValueError(f"compress: dtype must be float32 or float64, got {t.dtype}")
    t = t.contiguous()
    if t.data_ptr() % 16:
        t = t.clone()
    dt = "float32" if t.dtype == torch.float32 else "float64"
    dev = t.device.index if t.device.index is not None else torch.cuda.current_device()
    plan = plan_for(tuple(t.shape), 1, dt, dev)
    out = torch.empty_like(t)
    zeroed = torch.zeros(1, dtype=torch.int64, device=t.device)
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev)
        ws = torch.empty(plan.workspace_bytes, dtype=torch.uint8, device=t.device)
        scratch = torch.empty(plan.scratch_bytes, dtype=torch.uint8, device=t.device)  # per call (see force)
        plan.compress(t.data_ptr(), out.data_ptr(), float(epsilon), zeroed.data_ptr(), stream.cuda_stream,
                      ws.data_ptr(), scratch.data_ptr())
    total = t.numel()
    nz = int(zeroed.item())
    stats = {"total_coefficients": total, "zeroed_coefficients": nz, "zeroed_fraction": nz / total}
    return (out.cpu().numpy() if was_np else out), stats
