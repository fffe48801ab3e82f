"""Parity of the axis-0 1D transforms against the C oracle (developer tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle
import paper_2110_01172_b200 as sd

rng = np.random.default_rng(3)
worst = 0.0
for shape in [(8, 8), (16, 32), (256, 64), (64, 4096), (4096, 4), (1024, 8), (3, 64, 16)]:
    for dt in (torch.float64, torch.float32):
        if dt == torch.float32 and shape[-1] % 8:
            continue
        x = rng.uniform(-1, 1, shape)
        if dt == torch.float32:
            x = x.astype(np.float32).astype(np.float64)
        xt = torch.tensor(x, dtype=dt, device="cuda")
        y = sd.dct_axis0(xt).double().cpu().numpy()
        z = sd.idct_axis0(xt).double().cpu().numpy()
        xs = np.swapaxes(x, -1, -2)
        ry = np.swapaxes(oracle.port.dct_direct_1d(np.ascontiguousarray(xs)), -1, -2)
        rz = np.swapaxes(oracle.port.idct_direct_1d(np.ascontiguousarray(xs)), -1, -2)
        e1, e2 = oracle.rel_l2(y, ry), oracle.rel_l2(z, rz)
        if shape[-2] >= 4096:  # the direct O(N^2) oracle loses digits there: scipy's FFT-based DCT
            import scipy.fft as sf
            e1 = oracle.rel_l2(y, sf.dct(x, type=2, axis=-2) / 2)
            e2 = oracle.rel_l2(z, sf.dct(x, type=3, axis=-2) / 2)
        worst = max(worst, e1, e2) if dt == torch.float64 else worst
        print(shape, dt, f"dct {e1:.2e} idct {e2:.2e}", flush=True)
print("worst fp64", worst)
