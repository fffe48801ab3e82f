"""Host enqueue cost of plan.run vs device time per transform (developer tool).

1. enqueue-only: the GPU is held busy by a long sleep kernel, so the timed
   plan.run calls only measure the host side (pybind + maps + launches).
2. device: the same transforms captured in one CUDA graph and replayed,
   timed with events (no host in the loop)."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2110_01172_b200 as sd
from paper_2110_01172_b200 import _sdct

ap = argparse.ArgumentParser()
ap.add_argument("--size", type=int, nargs="+", default=[1024, 1024])
ap.add_argument("--dtype", default="float64")
ap.add_argument("--kinds", default="dct_2d,idct_2d")
ap.add_argument("--n", type=int, default=200)
a = ap.parse_args()
dt = torch.float64 if a.dtype == "float64" else torch.float32
shape = tuple(a.size)
rot = 8
xs = [torch.rand(shape, dtype=dt, device="cuda") for _ in range(rot)]
ys = [torch.empty_like(x) for x in xs]
plan = sd.plan_for(shape, 1, a.dtype, 0)
ws = torch.empty(plan.workspace_bytes, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
for kn in a.kinds.split(","):
    kind = getattr(_sdct, kn.upper())
    for i in range(10):
        plan.run(kind, xs[i % rot].data_ptr(), ys[i % rot].data_ptr(), s.cuda_stream, ws.data_ptr())
    torch.cuda.synchronize()
    torch.cuda._sleep(200_000_000)  # ~100 ms of GPU time
    t0 = time.perf_counter()
    for i in range(a.n):
        plan.run(kind, xs[i % rot].data_ptr(), ys[i % rot].data_ptr(), s.cuda_stream, ws.data_ptr())
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    host = (t1 - t0) / a.n * 1e6
    # graph-captured device time
    g = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    cs.wait_stream(s)
    with torch.cuda.stream(cs):
        with torch.cuda.graph(g, stream=cs):
            for i in range(a.n):
                plan.run(kind, xs[i % rot].data_ptr(), ys[i % rot].data_ptr(), cs.cuda_stream, ws.data_ptr())
    s.wait_stream(cs)
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(5):
        g.replay()
    e1.record(s)
    torch.cuda.synchronize()
    dev = e0.elapsed_time(e1) * 1e3 / (5 * a.n)
    # eager back-to-back (what bench's timed loop does)
    e0.record(s)
    for i in range(a.n):
        plan.run(kind, xs[i % rot].data_ptr(), ys[i % rot].data_ptr(), s.cuda_stream, ws.data_ptr())
    e1.record(s)
    torch.cuda.synchronize()
    eager = e0.elapsed_time(e1) * 1e3 / a.n
    print(f"{shape} {a.dtype} {kn}: host enqueue {host:6.2f} us/call | eager {eager:6.2f} us | graph {dev:6.2f} us")
