"""Quick parity check of the 4096-row fp64 column passes against the C oracle (developer tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle
import paper_2110_01172_b200 as sd

rng = np.random.default_rng(5)
for shape in [(4096, 4096), (4096, 64)]:
    x = rng.uniform(-1, 1, shape)
    xt = torch.tensor(x, device="cuda")
    y = sd.dct_2d(xt); torch.cuda.synchronize()
    print(shape, "dct_2d", oracle.rel_l2(y.cpu().numpy(), oracle.port.dct_2d(x)), flush=True)
    for k in ("idct_2d", "idct_idxst_2d", "idxst_idct_2d"):
        z = getattr(sd, k)(xt); torch.cuda.synchronize()
        print(shape, k, oracle.rel_l2(z.cpu().numpy(), getattr(oracle.port, k)(x)), flush=True)
xb = torch.tensor(rng.uniform(-1, 1, (3, 4096, 128)), device="cuda")
yb = sd.dct_2d(xb)
print("batch3 dct_2d", max(oracle.rel_l2(yb[i].cpu().numpy(), oracle.port.dct_2d(xb[i].cpu().numpy())) for i in range(3)))
