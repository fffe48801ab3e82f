"""Profiling driver: a few DCT->IDCT round trips at one size/dtype (for ncu)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2110_01172_b200 as sd
from paper_2110_01172_b200 import _sdct

ap = argparse.ArgumentParser()
ap.add_argument("--size", type=int, nargs="+", default=[4096, 4096])
ap.add_argument("--dtype", default="float64")
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--kinds", default="dct_2d,idct_2d")
a = ap.parse_args()
dt = torch.float64 if a.dtype == "float64" else torch.float32
shape = tuple(a.size)
x = torch.rand(shape, dtype=dt, device="cuda") * 2 - 1
plan = sd.plan_for(shape, 1, a.dtype, 0)
ws = torch.empty(plan.workspace_bytes, dtype=torch.uint8, device="cuda")
y = torch.empty_like(x); z = torch.empty_like(x)
s = torch.cuda.current_stream().cuda_stream
kinds = [getattr(_sdct, k.upper()) for k in a.kinds.split(",")]
for _ in range(a.iters):
    src, dst = x, y
    for k in kinds:
        plan.run(k, src.data_ptr(), dst.data_ptr(), s, ws.data_ptr())
        src, dst = dst, (z if dst is y else y)
torch.cuda.synchronize()
print("done")
