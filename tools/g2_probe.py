"""One generic-path 2D DCT + IDCT at a given shape (developer tool for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2110_01172_b200 as sd
n1, n2 = int(sys.argv[1]), int(sys.argv[2])
x = torch.rand((n1, n2), dtype=torch.float64, device="cuda")
for _ in range(2):
    y = sd.dct_2d(x)
    z = sd.idct_2d(y)
torch.cuda.synchronize()
