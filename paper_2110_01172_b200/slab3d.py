"""Slab-decomposed 3D DCT-II / IDCT over several GPUs.

One large 3D transform whose input is split along axis 0 across the ranks of a
process group (one process per GPU): rank r holds planes
[r*n1/G, (r+1)*n1/G) of x (n1, n2 divisible by G). The transform is separable
with the reference's unnormalised conventions (dct_3d = dctn/8,
proj/tests/python/test_smoke.py:46-50; dct_2d = dctn/4; dct_1d = dct/2), so

    dct_3d(x)  = dct_1d along axis 0  o  dct_2d over axes (1, 2)
    idct_3d(x) = idct_1d along axis 0 o  idct_2d over axes (1, 2)

and the slab pipeline is:

  1. local : batched 2D transform of this rank's planes (the fused fast path);
  2. all-to-all #1 (NCCL over NVLink): every rank sends rank t the columns
     j in t's axis-1 slab. Received as [src][i_loc][j_loc][k], which IS the
     (n1 x s2 n3) matrix with rows i = src s1 + i_loc in order — the axis-0
     placement falls out of the exchange, no reorder copy;
  3. local : the 1D transform along axis 0 of that matrix, taken in place by
     one persistent column pass (``dct_axis0`` / ``idct_axis0``,
     kernels_col1d.cuh: the axis-0 parity reorder rides on the tile load,
     the postprocess on the store) instead of transpose, contiguous 1D
     transform, transpose back;
  4. all-to-all #2: its output is already blocked by destination rank
     (rows t s1 .. t s1 + s1 - 1 are rank t's planes), so it is sent as is;
     the receiver's [src][i_loc][j_loc][k] becomes [i_loc][j][k] with one
     reorder copy.

Two full-tensor reorder copies per transform (the send blocks of #1 and the
final placement of #2) instead of the four of a transpose-based 1D leg. The
exchanges are the only collectives (the transposes are the "standard
communication operations" PAPER.md:649-660 mentions). The local transforms
are injectable so the exchange logic runs under gloo on CPU in tests/.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def _all_to_all(send: torch.Tensor, group) -> torch.Tensor:
    """Equal-split all-to-all of a contiguous [G, ...] tensor (block t goes to rank t)."""
    recv = torch.empty_like(send)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_to_all_single(recv, send, group=group)
    else:
        recv.copy_(send)
    return recv


def _slab_pipeline(x_local: torch.Tensor, n1: int, two_d, axis0, group) -> torch.Tensor:
    G = dist.get_world_size(group) if dist.is_initialized() else 1
    s1, n2, n3 = x_local.shape
    if s1 * G != n1 or n2 % G:
        raise ValueError(f"slab decomposition needs n1 = {s1}*{G} planes and n2 % {G} == 0")
    s2 = n2 // G
    # 1. 2D transform of every local plane (axes 1, 2)
    a = two_d(x_local.contiguous())                                   # [s1][n2][n3]
    # 2. block t = columns j of rank t's axis-1 slab: [G][s1][s2][n3]
    send = a.reshape(s1, G, s2, n3).permute(1, 0, 2, 3).contiguous()
    recv = _all_to_all(send, group)                                   # [G src][s1][s2][n3] = (n1 x s2 n3)
    # 3. 1D transform along axis 0 of the (n1 x s2 n3) matrix, in place of
    #    transpose + 1D + transpose
    c = axis0(recv.view(n1, s2 * n3))
    # 4. rows t*s1 .. t*s1+s1-1 are rank t's planes: already blocked by destination
    recv2 = _all_to_all(c.view(G, s1, s2, n3).contiguous(), group)   # [G src][s1][s2][n3]: j = src*s2 + j_loc
    return recv2.permute(1, 0, 2, 3).reshape(s1, n2, n3).contiguous()


def dct_3d_slab(x_local: torch.Tensor, n1: int, group=None, two_d=None, axis0=None) -> torch.Tensor:
    """This rank's axis-0 slab of dct_3d(x), given its slab of x (CUDA tensor,
    fp32/fp64). n1 is the global axis-0 extent (a power of two in [8, 4096]
    for the GPU axis-0 pass, with s2 n3 a multiple of 32 bytes' worth of
    elements). ``two_d`` / ``axis0`` replace the local transforms (tests)."""
    if two_d is None or axis0 is None:
        import paper_2110_01172_b200 as sd

        two_d = two_d or sd.dct_2d
        axis0 = axis0 or sd.dct_axis0
    return _slab_pipeline(x_local, n1, two_d, axis0, group)


def idct_3d_slab(x_local: torch.Tensor, n1: int, group=None, two_d=None, axis0=None) -> torch.Tensor:
    """This rank's axis-0 slab of idct_3d(x) (idct_3d(dct_3d(x)) = n1 n2 n3 / 8 x)."""
    if two_d is None or axis0 is None:
        import paper_2110_01172_b200 as sd

        two_d = two_d or sd.idct_2d
        axis0 = axis0 or sd.idct_axis0
    return _slab_pipeline(x_local, n1, two_d, axis0, group)
