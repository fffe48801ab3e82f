"""Generic-path probe (developer tool): parity + timing for large non-pow2 shapes."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle
import paper_2110_01172_b200 as sd

for shape in [(6000, 48), (48, 6000), (4100, 6), (5000, 4100)]:
    x = torch.rand(shape, dtype=torch.float64, device="cuda") * 2 - 1
    y = sd.dct_2d(x)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        y = sd.dct_2d(x)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) / 3 * 1e3
    err = None
    if shape[0] * shape[1] <= 400000:
        err = oracle.rel_l2(y.cpu().numpy(), oracle.port.dct_2d(x.cpu().numpy()))
    print(shape, f"{ms:.2f} ms", "rel_l2", err)
