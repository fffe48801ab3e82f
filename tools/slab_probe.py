"""Single-rank timing of the slab-decomposed 3D pipeline vs the fused 3D kernels (developer tool)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2110_01172_b200 as sd
from paper_2110_01172_b200 import slab3d

for shape, dt in [((256, 256, 256), torch.float32), ((128, 128, 128), torch.float64)]:
    x = torch.rand(shape, dtype=dt, device="cuda")
    for name, f in (("fused dct_3d", lambda: sd.dct_3d(x)), ("slab dct_3d", lambda: slab3d.dct_3d_slab(x, shape[0]))):
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            f()
        e1.record()
        torch.cuda.synchronize()
        print(shape, dt, name, f"{e0.elapsed_time(e1) / 10 * 1e3:.1f} us")
