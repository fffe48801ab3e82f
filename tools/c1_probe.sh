#!/bin/bash
# c1 (1024^2 fp64) latency probe: column-pass phase trace, per-stage times
# under band-width / PDL knobs, and the empty-kernel event floor.
set -x
python tools/trace_col.py 1024 float64
for nl in 2 4; do SDCT_FORCE_NL=$nl python tools/stage_time.py --size 1024 1024 --kinds dct_2d,idct_2d --reps 50; done
SDCT_NO_PDL=1 python tools/stage_time.py --size 1024 1024 --kinds dct_2d --reps 50
python - <<'PY'
import torch
x = torch.zeros(32, device="cuda"); s = torch.cuda.current_stream()
for n in (1, 2):
    ts = []
    for r in range(50):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(n): x.add_(1)
        e1.record(s); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    ts.sort(); print(f"{n} tiny kernels between events: {ts[25]*1e3:.1f} us")
PY
