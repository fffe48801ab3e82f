"""Host-side cost per call vs GPU time (developer tool): is a workload launch-bound?"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2110_01172_b200 as sd
from paper_2110_01172_b200 import _sdct

for shape, dt, mode in [((2048, 2048), "float64", "force"), ((1024, 1024), "float64", "dct"), ((4096, 4096), "float64", "rt"),
                        ((256, 256, 256), "float32", "dct3")]:
    tdt = torch.float64 if dt == "float64" else torch.float32
    x = torch.rand(shape, dtype=tdt, device="cuda")
    o1, o2 = torch.empty_like(x), torch.empty_like(x)
    plan = sd.plan_for(shape, 1, dt, 0)
    ws = torch.empty(plan.workspace_bytes, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    def step():
        if mode == "force":
            plan.force_fields(x.data_ptr(), o1.data_ptr(), o2.data_ptr(), s, ws.data_ptr())
        elif mode == "dct":
            plan.run(_sdct.DCT_2D, x.data_ptr(), o1.data_ptr(), s, ws.data_ptr())
        elif mode == "dct3":
            plan.run(_sdct.DCT_3D, x.data_ptr(), o1.data_ptr(), s, ws.data_ptr())
        else:
            plan.run(_sdct.DCT_2D, x.data_ptr(), o1.data_ptr(), s, ws.data_ptr())
            plan.run(_sdct.IDCT_2D, o1.data_ptr(), o2.data_ptr(), s, ws.data_ptr())
    for _ in range(20):
        step()
    torch.cuda.synchronize()
    n = 200
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(n):
        step()
    t1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{mode} {shape} {dt}: host issue {1e6*(t1-t0)/n:.1f} us/step, gpu {1e3*e0.elapsed_time(e1)/n:.1f} us/step, wall {1e6*(t2-t0)/n:.1f}")
    # host-only cost: the same step with the GPU busy in a long kernel
    torch.cuda._sleep(200_000_000)
    t0 = time.perf_counter()
    for _ in range(50):
        step()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"   host issue with queue backed up: {1e6*(t1-t0)/50:.1f} us/step")
