"""Per-stage kernel times (CUDA events, L2 flushed before each launch) of the
DCT / IDCT pipelines at one size; developer tool for A/B runs of env knobs."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2110_01172_b200 as sd
from paper_2110_01172_b200 import _sdct

ap = argparse.ArgumentParser()
ap.add_argument("--size", type=int, nargs="+", default=[4096, 4096])
ap.add_argument("--dtype", default="float64")
ap.add_argument("--kinds", default="dct_2d,idct_2d")
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
dt = torch.float64 if a.dtype == "float64" else torch.float32
shape = tuple(a.size)
x = torch.rand(shape, dtype=dt, device="cuda") * 2 - 1
plan = sd.plan_for(shape, 1, a.dtype, 0)
ws = torch.empty(plan.workspace_bytes, dtype=torch.uint8, device="cuda")
y = torch.empty_like(x)
s = torch.cuda.current_stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
nbytes = 2 * x.numel() * x.element_size()
out = []
for kn in a.kinds.split(","):
    kind = getattr(_sdct, kn.upper())
    plan.run(kind, x.data_ptr(), y.data_ptr(), s.cuda_stream, ws.data_ptr())
    for st in range(plan.stage_count(kind)):
        ts = []
        for r in range(a.reps):
            flush.fill_(r & 255)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            plan.run_stage(kind, st, x.data_ptr(), y.data_ptr(), s.cuda_stream, ws.data_ptr())
            e1.record(s)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts = sorted(ts[2:])
        med = ts[len(ts) // 2]
        out.append(f"{kn}.{st} {med * 1e3:7.1f} us {nbytes / med / 1e6:7.0f} GB/s")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for r in range(a.reps):
        plan.run(kind, x.data_ptr(), y.data_ptr(), s.cuda_stream, ws.data_ptr())
    e1.record(s)
    torch.cuda.synchronize()
    out.append(f"{kn} full (back-to-back) {e0.elapsed_time(e1) / a.reps * 1e3:7.1f} us")
print(" | ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("SDCT_")), a.dtype, shape)
print("\n".join(out))
