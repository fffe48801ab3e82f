"""Quick GPU parity sweep (developer tool): every transform kind x dtype x shape
against the C oracle. Prints rel-L2 per case."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
import paper_2110_01172_b200 as sd

rng = np.random.default_rng(7)
shapes2 = [(8, 8), (2, 8), (4, 16), (16, 8), (64, 64), (32, 128), (256, 256), (1024, 1024), (4096, 4096), (7, 9), (33, 17), (16, 3), (1, 1)]
shapes3 = [(2, 2, 8), (4, 4, 8), (8, 16, 32), (16, 8, 16), (64, 64, 64), (3, 4, 5), (5, 6, 7)]
kinds2 = ["dct_2d", "idct_2d", "idct_idxst_2d", "idxst_idct_2d"]
kinds3 = ["dct_3d", "idct_3d"]
worst = {}
for dt in (torch.float64, torch.float32):
    for shapes, kinds in ((shapes2, kinds2), (shapes3, kinds3)):
        for shp in shapes:
            x = rng.uniform(-1, 1, shp)
            if dt == torch.float32:
                x = x.astype(np.float32).astype(np.float64)
            xt = torch.tensor(x, dtype=dt, device="cuda")
            for k in kinds:
                if max(shp) >= 4096 and k not in ("dct_2d", "idct_2d"):
                    continue
                y = getattr(sd, k)(xt)
                torch.cuda.synchronize()
                want = getattr(oracle.port, k)(x)
                e = oracle.rel_l2(y.double().cpu().numpy(), want)
                tag = f"{k} {shp} {str(dt)[6:]}"
                print(f"{tag:40s} rel_l2={e:.3e}", flush=True)
                worst[str(dt)] = max(worst.get(str(dt), 0), e)
print("worst", worst)
# numpy drop-in path
x = rng.uniform(-1, 1, (64, 48))
print("numpy dct_2d", oracle.rel_l2(sd.dct_2d(x), oracle.port.dct_2d(x)))
print("numpy idct_3d", oracle.rel_l2(sd.idct_3d(rng.uniform(-1,1,(8,8,8))), 0) if False else "skip")
