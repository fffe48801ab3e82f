"""One 3D generic-path transform for an ncu launch list (developer tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2110_01172_b200 as sd
s = tuple(int(v) for v in sys.argv[1].split("x"))
x = torch.rand(s, dtype=torch.float64, device="cuda")
sd.dct_3d(x); torch.cuda.synchronize()
y = sd.dct_3d(x); torch.cuda.synchronize()
