"""Wall time of the reference-surface numpy calls (developer tool)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2110_01172_b200 as sd

for n in (1024, 4096):
    x = np.random.default_rng(0).uniform(-1, 1, (n, n))
    y = sd.idct_2d(sd.dct_2d(x))
    for rep in range(2):
        t0 = time.perf_counter(); y1 = sd.dct_2d(x); t1 = time.perf_counter(); y2 = sd.idct_2d(y1); t2 = time.perf_counter()
    out = np.empty_like(x)
    t3 = time.perf_counter(); out[...] = x; t4 = time.perf_counter()
    print(f"{n}^2: dct_2d {1e3*(t1-t0):.1f} ms, idct_2d {1e3*(t2-t1):.1f} ms, rel err {np.linalg.norm(y2/(n*n/4)-x)/np.linalg.norm(x):.1e}; host memcpy {1e3*(t4-t3):.1f} ms")
