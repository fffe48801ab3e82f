"""3D generic-path timing against cuFFT rfftn/irfftn of the same shape (developer tool)."""
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
    (200, 200, 200), (250, 250, 250), (255, 255, 255), (100, 120, 130), (256, 256, 250), (97, 101, 103)]
for dt in (torch.float64, torch.float32):
    for s in shapes:
        x = torch.rand(s, dtype=dt, device="cuda")
        a = t(lambda: sd.dct_3d(x))
        b = t(lambda: sd.idct_3d(x))
        c = t(lambda: torch.fft.rfftn(x))
        X = torch.fft.rfftn(x)
        d = t(lambda: torch.fft.irfftn(X, s=s))
        gb = 2 * x.numel() * x.element_size() / 1e3
        print(f"{str(dt)[6:]:8s} {s!s:16s} dct3 {a:8.1f} us ({gb / a:6.0f} GB/s) vs rfftn {c:8.1f} ({a / c:4.2f}x) | "
              f"idct3 {b:8.1f} vs irfftn {d:8.1f} ({b / d:4.2f}x)")
