"""Profiling driver: a few force_demo_fields steps at one size/dtype (for ncu),
plus graph-timed paired vs unpaired steps when run without ncu."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2110_01172_b200 as sd

ap = argparse.ArgumentParser()
ap.add_argument("--size", type=int, nargs="+", default=[2048, 2048])
ap.add_argument("--dtype", default="float64")
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--time", action="store_true")
a = ap.parse_args()
dt = torch.float64 if a.dtype == "float64" else torch.float32
shape = tuple(a.size)
xs = [torch.rand(shape, dtype=dt, device="cuda") * 2 - 1 for _ in range(6)]
plan = sd.plan_for(shape, 1, a.dtype, 0)
ws = torch.empty(plan.workspace_bytes, dtype=torch.uint8, device="cuda")
o1 = torch.empty_like(xs[0]); o2 = torch.empty_like(xs[0])
s = torch.cuda.current_stream()
for i in range(a.iters):
    plan.force_fields(xs[i % 6].data_ptr(), o1.data_ptr(), o2.data_ptr(), s.cuda_stream, ws.data_ptr())
torch.cuda.synchronize()
if a.time:
    import bench
    for env in ("0", "1"):
        os.environ["SDCT_FORCE_UNPAIRED"] = env
        ms, ok = bench.graph_time(lambda sh, j=[0]: (plan.force_fields(xs[j[0] % 6].data_ptr(), o1.data_ptr(),
                                                                      o2.data_ptr(), sh, ws.data_ptr()),
                                                    j.__setitem__(0, j[0] + 1)), 60, s)
        print(f"unpaired={env} force step {ms * 1e3:.1f} us (graph={ok})")
print("done")
