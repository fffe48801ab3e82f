"""Regenerate profiles/r02_c2_f64.md: ncu summary of the c2 fp64 kernels plus
the live roofline table from profiles/r02/bench_c2.json (developer tool)."""
import json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep, launches = sys.argv[1], sys.argv[2]
out = os.path.join(ROOT, "profiles", "r02_c2_f64")
subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep, out, "--launches", launches,
                "--stage-map", "dct_2d.stage0=a;dct_2d.stage1=b;idct_2d.stage0=c;idct_2d.stage1=d",
                "--traffic-prefix", "c2:float64:"], check=True, capture_output=True)
b = json.load(open(os.path.join(ROOT, "profiles", "r02", "bench_c2.json")))
peak = b["roofline"]["peak"]
names = {"dct_2d.stage0": "col fwd `col_kernel<double,4096,2,0,0,0>`", "dct_2d.stage1": "row fwd `rowp_kernel<double,2048,0>`",
         "idct_2d.stage0": "row inv `rowp_kernel<double,2048,1>`", "idct_2d.stage1": "col inv `col_kernel<double,4096,2,1,1,1>`"}
r01 = {"dct_2d.stage0": 86.1, "dct_2d.stage1": 71.9, "idct_2d.stage0": 87.7, "idct_2d.stage1": 78.5}
rows = [f"| {names[k['kernel']]} | {r01[k['kernel']]:.1f} | {k['ms'] * 1e3:.1f} | {k['gbs']:.0f} | {k['gbs'] / peak:.3f} |"
        for k in b["roofline"]["all_kernels"]]
txt = open(out + ".md").read()
txt += f"""
## Round 2: live per-kernel roofline (bench.py c2, `profiles/r02/bench_c2.json`)

Algorithmic bytes per launch = 2 * 4096^2 * 8 = 268,435,456 B; peak = MEASURED_PEAKS.json
hbm_gbs = {peak} GB/s. Live times: per-kernel CUDA graphs (50 back-to-back launches of each kernel on the timed loop's rotating buffers, events around the replay).

| kernel | r01 us | r02 us | GB/s | frac |
|---|---|---|---|---|
""" + "\n".join(rows) + f"""

Step (PDL, back to back): {b['ms_per_step'] * 1e3:.1f} us (round 1: 307.6 us); value {b['value']} GB/s;
round-trip parity {b['parity']['round_trip_rel_l2']:.2e}, forward vs the C oracle
{b['parity'].get('dct_2d_rel_l2_vs_oracle', float('nan')):.2e}.

What changed since round 1:
* col fwd: the next tile's TMA load is issued right after the stage-0 operands are read; the two
  exchanges run through the 64 KB staging buffer in balanced half rounds (CTA-wide, then
  warp-local). Its data-movement floor (the same schedule without the FFT, `tools/microbench_xs.cu`)
  is 57.8 us = 0.71 of peak; the kernel spends 9.3 us per tile against that floor's 8.35 us.
* row fwd / row inv: `rowp_kernel` (kernels_rowp.cuh) - mirror-paired radix-8 stage (lane and
  lane^16 own the frequency sets k and M-k), postprocess / preprocess+packing from registers after
  one shuffle exchange, per-thread twiddle bases times compile-time steps, per-item table loads
  issued ahead of the waits they overlap; the inverse on the persistent ring (DIT) with coalesced
  32-B-sector stores straight from registers.
* ncu DRAM bytes per launch stay at or below the 268 MB algorithmic figure: no re-reads.
"""
open(out + ".md", "w").write(txt)
print(out + ".md")
