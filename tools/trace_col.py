"""Phase trace of the persistent column kernel (developer tool).

Uses the debug hook sdct_debug_set_trace (8 u64 per tile: loop start, tile
landed, next load issued, [early-reissue schedule: CTA-wide exchange done,
warp exchange done, last stage done], stores issued, CTA id)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2110_01172_b200 as sd
from paper_2110_01172_b200 import _sdct, capi

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
dt = sys.argv[2] if len(sys.argv) > 2 else "float64"
tdt = torch.float64 if dt == "float64" else torch.float32
x = torch.rand((n, n), dtype=tdt, device="cuda")
plan = sd.plan_for((n, n), 1, dt, 0)
ws = torch.empty(plan.workspace_bytes, dtype=torch.uint8, device="cuda")
y = torch.empty_like(x)
s = torch.cuda.current_stream().cuda_stream
tr = torch.zeros(8 * 65536, dtype=torch.int64, device="cuda")
lib = capi.lib()
lib.sdct_debug_set_trace.argtypes = [ctypes.c_void_p]
for kind, st in ((_sdct.DCT_2D, 0), (_sdct.IDCT_2D, 1)):
    for rep in range(3):
        lib.sdct_debug_set_trace(tr.data_ptr() if rep == 2 else None)
        tr.zero_()
        plan.run_stage(kind, st, x.data_ptr(), y.data_ptr(), s, ws.data_ptr())
        torch.cuda.synchronize()
    lib.sdct_debug_set_trace(None)
    a = tr.view(-1, 8).cpu().numpy()
    a = a[a[:, 0] > 0]
    t0 = a[:, 0].min()
    tot = (a[:, 6].max() - t0) / 1e3
    ctas = sorted(set(a[:, 7].tolist()))
    print(f"{dt} kind {kind}: tiles {len(a)}  span {tot:.1f} us  ctas {len(ctas)}")
    print(f"  wait for tile        mean {((a[:, 1] - a[:, 0]) / 1e3).mean():.2f} us")
    print(f"  landed -> next issued mean {((a[:, 2] - a[:, 1]) / 1e3).mean():.2f} us")
    if (a[:, 3] > 0).all():
        print(f"  -> CTA exchange done  mean {((a[:, 3] - a[:, 2]) / 1e3).mean():.2f} us")
        print(f"  -> warp exchange done mean {((a[:, 4] - a[:, 3]) / 1e3).mean():.2f} us")
        print(f"  -> last stage done    mean {((a[:, 5] - a[:, 4]) / 1e3).mean():.2f} us")
        print(f"  -> stores issued      mean {((a[:, 6] - a[:, 5]) / 1e3).mean():.2f} us")
    else:
        print(f"  -> stores issued      mean {((a[:, 6] - a[:, 2]) / 1e3).mean():.2f} us")
