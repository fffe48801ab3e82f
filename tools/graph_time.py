"""Graph-timed transform calls (developer A/B tool): CUDA graph of N calls of
one kind on rotating inputs (past L2), replayed, events around the replay."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2110_01172_b200 import _sdct

ap = argparse.ArgumentParser()
ap.add_argument("--size", type=int, nargs="+", default=[1024, 1024])
ap.add_argument("--dtype", default="float64")
ap.add_argument("--kinds", default="dct_2d")
ap.add_argument("--reps", type=int, default=100)
a = ap.parse_args()
dt = torch.float64 if a.dtype == "float64" else torch.float32
shape = tuple(a.size)
nb = max(1, (300 << 20) // (2 * torch.tensor([], dtype=dt).element_size() * int(torch.tensor(shape).prod())))
xs = [torch.rand(shape, dtype=dt, device="cuda") * 2 - 1 for _ in range(nb)]
ys = [torch.empty_like(xs[0]) for _ in range(nb)]
plan = _sdct.Plan(list(shape), 1, a.dtype)
ws = torch.empty(plan.workspace_bytes, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
for kn in a.kinds.split(","):
    k = getattr(_sdct, kn.upper())
    def one(sh, j=[0]):
        r = j[0] % nb
        j[0] += 1
        plan.run(k, xs[r].data_ptr(), ys[r].data_ptr(), sh, ws.data_ptr())
    ms, ok = bench.graph_time(one, a.reps, s)
    print(" ".join(f"{k_}={v}" for k_, v in os.environ.items() if k_.startswith("SDCT_")), a.dtype, shape, kn,
          f"{ms * 1e3:.2f} us (graph={ok}, {nb} rotating buffers)")
