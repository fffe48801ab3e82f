"""e2e probe (developer tool): stream_host throughput for small items + host enqueue cost."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2110_01172_b200 as sd

for n in (1024, 2048):
    x = (torch.rand((1, n, n), dtype=torch.float64) * 2 - 1).pin_memory()
    o = torch.empty_like(x).pin_memory()
    s = torch.cuda.current_stream()
    sd.stream_host(["dct_2d"], x, o, count=4)
    torch.cuda.synchronize()
    for cnt in (50, 200):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(s)
        sd.stream_host(["dct_2d"], x, o, count=cnt, sync=False)
        t1 = time.perf_counter()
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / cnt
        print(f"n={n} count={cnt}: {ms * 1e3:7.1f} us/item on device, host enqueue {(t1 - t0) / cnt * 1e6:6.1f} us/item, "
              f"e2e {2 * n * n * 8 / ms / 1e6:6.1f} GB/s")
