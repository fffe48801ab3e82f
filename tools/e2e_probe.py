"""e2e probe (developer tool): stream_host throughput at 4096^2 fp64 vs chain."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2110_01172_b200 as sd

n = 4096
x = (torch.rand((1, n, n), dtype=torch.float64) * 2 - 1).pin_memory()
o = torch.empty_like(x).pin_memory()
xs = (torch.rand((8, n, n), dtype=torch.float64) * 2 - 1).pin_memory()
os_ = torch.empty_like(xs).pin_memory()
s = torch.cuda.current_stream()
for chain in (["dct_2d"], ["dct_2d", "idct_2d"]):
    for name, xi, oi, cnt in (("same-buffers", x, o, 40), ("distinct-8", xs, os_, 8)):
        sd.stream_host(chain, xi, oi, count=cnt if xi.shape[0] == 1 else None)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        sd.stream_host(chain, xi, oi, count=cnt if xi.shape[0] == 1 else None, sync=False)
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / cnt
        print(f"{'+'.join(chain):16s} {name:13s} {ms:6.3f} ms/item  {2 * n * n * 8 / ms / 1e6:6.1f} GB/s PCIe per direction")
