"""Small transforms of every kernel family for compute-sanitizer runs (developer tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2110_01172_b200 as sd

torch.manual_seed(0)
for dt in (torch.float64, torch.float32):
    # (4096, 64): early-reissue fp64 column pass; (64, 4096) / (32, 2048) / batched:
    # the mirror-paired row kernels (M = 2048 / 1024)
    for shape in [(64, 128), (2048, 2048), (16, 4096), (4096, 64), (64, 4096), (32, 2048), (2, 64, 4096)]:
        x = torch.rand(shape, dtype=dt, device="cuda")
        for f in (sd.dct_2d, sd.idct_2d, sd.idct_idxst_2d, sd.idxst_idct_2d):
            f(x)
        sd.force_demo_fields(x)
        if x.dim() == 2:
            sd.compress(x, 0.5)
    x3 = torch.rand((16, 8, 32), dtype=dt, device="cuda")
    sd.dct_3d(x3)
    sd.idct_3d(x3)
    sd.dct_2d(torch.rand((7, 9), dtype=dt, device="cuda"))
    # generic two-pass 2D pipeline: both tile configurations, odd / prime extents, batch
    for shape in [(100, 60), (33, 17), (3, 2500), (2500, 3), (97, 101), (2, 50, 30)]:
        xg = torch.rand(shape, dtype=dt, device="cuda")
        for f in (sd.dct_2d, sd.idct_2d, sd.idct_idxst_2d, sd.idxst_idct_2d):
            f(xg)
    sd.dct_2d(torch.rand((8192, 16), dtype=dt, device="cuda"))
    # axis-0 column pass (slab3d's axis-0 leg)
    xa = torch.rand((2, 256, 64), dtype=dt, device="cuda")
    sd.dct_axis0(xa)
    sd.idct_axis0(xa)
torch.cuda.synchronize()
print("probe done")
