"""Generic-path (non-power-of-two) timing against cuFFT R2C/C2R of the same
shape (torch.fft, which calls cuFFT) — developer tool."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2110_01172_b200 as sd


def t(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


shapes = [tuple(int(v) for v in a.split("x")) for a in sys.argv[1:]] or [
    (1000, 1000), (1536, 1536), (2000, 2000), (3000, 3000), (3072, 3072), (4095, 4095), (1023, 1023),
    (4097, 4097), (2048, 3000), (6000, 6000)]
for dt in (torch.float64, torch.float32):
    for s in shapes:
        x = torch.rand(s, dtype=dt, device="cuda")
        fast = sd.plan_for(s, 1, "float64" if dt == torch.float64 else "float32", 0).fast
        a = t(lambda: sd.dct_2d(x))
        b = t(lambda: sd.idct_2d(x))
        c = t(lambda: torch.fft.rfft2(x))
        X = torch.fft.rfft2(x)
        d = t(lambda: torch.fft.irfft2(X, s=s))
        gb = 2 * x.numel() * x.element_size() / 1e3
        print(f"{str(dt)[6:]:8s} {s!s:14s} fast={int(fast)} dct {a:8.1f} us ({gb / a:6.0f} GB/s) vs R2C {c:8.1f} "
              f"({a / c:4.2f}x) | idct {b:8.1f} vs C2R {d:8.1f} ({b / d:4.2f}x)")
