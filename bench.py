#!/usr/bin/env python
"""Benchmark of the hot path: 2D DCT -> IDCT round trip at 4096^2 fp64
(BASELINE.json configs[1], the configuration the headline metric is quoted on).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--size 4096] [--dtype float64|float32]

One step = dct_2d then idct_2d of one 4096x4096 fp64 image (inputs resident
in HBM for `value`). Algorithmic bytes per transform = 2 * numel * sizeof(T)
(read the input once, write the output once), so a step moves
4 * numel * sizeof(T) algorithmic bytes. Working set per step (input, DCT
output, IDCT output, workspace = 4 x 134 MB) is > 4x the 126 MB L2, so no step
re-reads the previous step's data from L2.

N > 1 (torchrun): every rank transforms its own image (independent objects,
no data-path collective) -> weak scaling; value = all ranks' bytes / max-over-
ranks time. Rank 0 prints one JSON line.

--impl reference: the unmodified reference CPU library (oracle/_ref, built from
/root/reference by oracle/Makefile) on this host's cores, same metric/unit.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "2D DCT/IDCT ms & effective GB/s at 4096² fp64 vs HBM roofline & CPU ref"
UNIT = "GB/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _cores():
    n = len(os.sched_getaffinity(0))
    quota = None
    try:
        with open("/sys/fs/cgroup/cpu.max") as f:
            q, per = f.read().split()
            if q != "max":
                quota = float(q) / float(per)
    except Exception:
        pass
    return n, quota


class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons during timing."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() in ("active", "1", "yes"):
                    reasons.add(nm)
        loaded = [s for s in sm if mx and s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
def cpu_reference_rate(n: int, budget_s: float, max_steps: int | None = None):
    """Round trips of the reference (oracle/_ref, all host threads) on an n x n
    fp64 image; returns (GB/s, seconds per round trip, round trips timed, kind)."""
    import numpy as np

    import oracle

    x = np.random.default_rng(2).uniform(-1.0, 1.0, size=(n, n))
    if oracle.ref_available():
        kind = "reference"
        fwd = lambda a: oracle.ref.run("dct_2d", a, threads=0)  # noqa: E731
        inv = lambda a: oracle.ref.run("idct_2d", a, threads=0)  # noqa: E731
    else:
        kind = "port"
        fwd, inv = oracle.port.dct_2d, oracle.port.idct_2d
    t0 = time.perf_counter()
    inv(fwd(x))  # warm-up round trip (also sizes the sample)
    t_rt = time.perf_counter() - t0
    steps = max(1, int(budget_s / max(t_rt, 1e-3)))
    if max_steps is not None:
        steps = min(steps, max_steps)
    t0 = time.perf_counter()
    for _ in range(steps):
        inv(fwd(x))
    dt = (time.perf_counter() - t0) / steps
    bytes_rt = 4.0 * n * n * 8
    return bytes_rt / dt / 1e9, dt, steps, kind


# ---------------------------------------------------------------------------
def cufft_times(x, n, stream, reps):
    """cuFFT R2C and C2R (D2Z / Z2D for fp64) of the same n x n shape, called
    directly through libcufft (ctypes) so no framework copies or plan-cache
    effects are timed. Library baseline only (north_star: 'cuFFT R2C on the
    same shape ... reported alongside'). Returns (r2c_ms, c2r_ms)."""
    import ctypes

    import torch

    lib = None
    for name in ("libcufft.so.11", "libcufft.so"):
        try:
            lib = ctypes.CDLL(name)
            break
        except OSError:
            continue
    if lib is None:
        raise RuntimeError("libcufft not loadable")
    f64 = x.dtype == torch.float64
    fwd_type, inv_type = (0x6A, 0x6C) if f64 else (0x2A, 0x2C)
    spec = torch.empty((n, n // 2 + 1), dtype=torch.complex128 if f64 else torch.complex64, device=x.device)
    out = torch.empty_like(x)
    pf, pi = ctypes.c_int(0), ctypes.c_int(0)
    assert lib.cufftPlan2d(ctypes.byref(pf), n, n, fwd_type) == 0
    assert lib.cufftPlan2d(ctypes.byref(pi), n, n, inv_type) == 0
    sp = ctypes.c_void_p(stream.cuda_stream)
    lib.cufftSetStream(pf, sp)
    lib.cufftSetStream(pi, sp)
    exf = lib.cufftExecD2Z if f64 else lib.cufftExecR2C
    exi = lib.cufftExecZ2D if f64 else lib.cufftExecC2R
    xi, so, oo = ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(spec.data_ptr()), ctypes.c_void_p(out.data_ptr())
    res = []
    for ex, a_, b_ in ((exf, xi, so), (exi, so, oo)):
        for _ in range(3):
            assert ex(pf if ex is exf else pi, a_, b_) == 0
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            ex(pf if ex is exf else pi, a_, b_)
        e1.record(stream)
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) / reps)
    lib.cufftDestroy(pf)
    lib.cufftDestroy(pi)
    return res[0], res[1]



def run_reference(args, rank: int):
    if rank != 0:
        return
    n = args.size
    # bound the whole --steps K --warmup W run to a few minutes of CPU time
    rate, dt, steps, kind = cpu_reference_rate(n, budget_s=150.0, max_steps=args.steps)
    cores, quota = _cores()
    line = {
        "impl": "reference", "metric": METRIC, "value": round(rate, 4), "unit": UNIT,
        "n_gpus": args.gpus, "steps": steps, "warmup": 1, "ms_per_step": round(dt * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic uniform(-1,1)",
        "config": {"workload": f"2D DCT-II -> IDCT round trip {n}x{n} fp64 (BASELINE configs[1])",
                   "requested_steps": args.steps, "requested_warmup": args.warmup},
        "cpu_baseline": {"value": round(rate, 4), "unit": UNIT, "cores": cores, "kind": kind,
                         "cgroup_cpu_quota": quota,
                         "sample": f"{steps} round trips of dct_2d+idct_2d {n}x{n} fp64, prebuilt plans, threads=0"},
        "e2e": {"value": round(rate, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def run_ours(args, rank: int, world: int, local_rank: int):
    import torch
    import torch.distributed as dist

    import paper_2110_01172_b200 as sd
    from paper_2110_01172_b200 import _sdct

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    n = args.size
    dt = torch.float64 if args.dtype == "float64" else torch.float32
    esz = 8 if dt == torch.float64 else 4
    numel = n * n
    bytes_transform = 2.0 * numel * esz
    bytes_step = 2 * bytes_transform

    g = torch.Generator(device="cpu").manual_seed(2 + rank)
    x_host = (torch.rand((n, n), generator=g, dtype=torch.float64) * 2 - 1).to(dt)
    x = x_host.to(dev)
    stream = torch.cuda.current_stream(dev)

    plan = sd.plan_for((n, n), 1, args.dtype, local_rank)
    ws = torch.empty(plan.workspace_bytes, dtype=torch.uint8, device=dev)
    y = torch.empty_like(x)
    z = torch.empty_like(x)
    s = stream.cuda_stream

    def step():
        plan.run(_sdct.DCT_2D, x.data_ptr(), y.data_ptr(), s, ws.data_ptr())
        plan.run(_sdct.IDCT_2D, y.data_ptr(), z.data_ptr(), s, ws.data_ptr())

    def barrier():
        if world > 1:
            dist.barrier()

    # parity spot check of this rank's own data (round trip = N1 N2 / 4 x)
    step()
    torch.cuda.synchronize()
    rt_err = float(((z / (numel / 4.0) - x).norm() / x.norm()).item())

    clocks = ClockSampler(local_rank)
    clocks.start()
    t_w = time.perf_counter()
    i = 0
    while i < args.warmup or time.perf_counter() - t_w < 1.0:  # >= W steps and >= 1 s soak
        step()
        i += 1
        if i % 50 == 0:
            torch.cuda.synchronize()
    warm_done = i
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms = e0.elapsed_time(e1)
    clk = clocks.stop()
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    value = world * bytes_step * args.steps / (ms / 1e3) / 1e9

    # ---- per-kernel timing (roofline of the dominant kernel) ----------------
    peak, peak_kind = _peaks()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    kernels = []
    for kind_name, kind, src, dst in (("dct_2d", _sdct.DCT_2D, x, y), ("idct_2d", _sdct.IDCT_2D, y, z)):
        for st in range(plan.stage_count(kind)):
            times = []
            for _ in range(10):
                flush.fill_(1)  # evict L2 (256 MB > 126 MB) outside the timed launch
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                plan.run_stage(kind, st, src.data_ptr(), dst.data_ptr(), s, ws.data_ptr())
                b.record(stream)
                torch.cuda.synchronize()
                times.append(a.elapsed_time(b))
            avg = sum(times[2:]) / len(times[2:])
            kernels.append({"kernel": f"{kind_name}.stage{st}", "ms": avg,
                            "gbs": bytes_transform / (avg / 1e3) / 1e9})
        # re-run the full transform so dst holds valid data for the next kind
        plan.run(kind, src.data_ptr(), dst.data_ptr(), s, ws.data_ptr())
    torch.cuda.synchronize()
    dom = max(kernels, key=lambda k: k["ms"])
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            traffic = json.load(f).get(dom["kernel"])
    except Exception:
        pass
    roofline = {"bound": "hbm", "achieved": round(dom["gbs"], 2), "peak": peak, "unit": "GB/s",
                "frac": round(dom["gbs"] / peak, 4), "traffic": traffic, "kernel": dom["kernel"],
                "peak_kind": peak_kind,
                "per_launch_bytes": bytes_transform,
                "all_kernels": [{k2: (round(v, 4) if isinstance(v, float) else v) for k2, v in k.items()}
                                for k in kernels],
                "step_frac": round(value / world / peak, 4),
                "step_frac_2pass_normalised": round(2 * value / world / peak, 4)}

    # ---- cuFFT on the same shape (library baseline, reported alongside) -----
    cufft = {}
    try:
        reps = 20
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        r2c, c2r = cufft_times(x, n, stream, reps)
        ours = {}
        for kn, kind, src, dst in (("dct", _sdct.DCT_2D, x, y), ("idct", _sdct.IDCT_2D, y, z)):
            a.record(stream)
            for _ in range(reps):
                plan.run(kind, src.data_ptr(), dst.data_ptr(), s, ws.data_ptr())
            b.record(stream)
            torch.cuda.synchronize()
            ours[kn] = a.elapsed_time(b) / reps
        cufft = {"api": "libcufft cufftPlan2d + cufftExec{D2Z,Z2D|R2C,C2R}, plan built outside timing",
                 "r2c_ms": round(r2c, 4), "c2r_ms": round(c2r, 4), "dct_ms": round(ours["dct"], 4),
                 "idct_ms": round(ours["idct"], 4), "dct_over_r2c": round(ours["dct"] / r2c, 3),
                 "idct_over_c2r": round(ours["idct"] / c2r, 3)}
    except Exception as e:  # pragma: no cover - reported, not fatal
        cufft = {"error": str(e)}

    # ---- end to end through the public API with host buffers ---------------
    x_pin = x_host.pin_memory()
    out_pin = torch.empty_like(x_pin).pin_memory()
    xd = torch.empty_like(x)

    def e2e_step():
        xd.copy_(x_pin, non_blocking=True)
        yy = sd.dct_2d(xd)
        zz = sd.idct_2d(yy)
        out_pin.copy_(zz, non_blocking=True)

    for _ in range(3):
        e2e_step()
    torch.cuda.synchronize()
    barrier()
    e_steps = max(5, min(args.steps, 50))
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(e_steps):
        e2e_step()
    b.record(stream)
    torch.cuda.synchronize()
    e_ms = a.elapsed_time(b)
    if world > 1:
        t = torch.tensor([e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_ms = float(t.item())
    e2e_val = world * bytes_step * e_steps / (e_ms / 1e3) / 1e9
    e2e_err = float(((out_pin.to(torch.float64) / (numel / 4.0) - x_host.to(torch.float64)).norm()
                     / x_host.to(torch.float64).norm()).item())

    # ---- CPU baseline (rank 0, N = 1 only) -----------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        rate, dtr, steps, kind = cpu_reference_rate(n, budget_s=args.cpu_budget)
        cores, quota = _cores()
        cpu = {"value": round(rate, 4), "unit": UNIT, "cores": cores, "kind": kind,
               "cgroup_cpu_quota": quota,
               "sample": f"{steps} round trips of dct_2d+idct_2d {n}x{n} fp64 on the host, prebuilt plans, "
                         f"threads=0 ({dtr * 1e3:.1f} ms each)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": warm_done, "ms_per_step": round(ms_per_step, 5),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64" if dt == torch.float64 else "f32",
            "data": "synthetic uniform(-1,1), device-resident",
            "config": {"workload": f"2D DCT-II -> IDCT round trip {n}x{n} {args.dtype} per GPU (BASELINE configs[1])",
                       "global_batch": world, "parallelism": f"replicas x{world} (independent images, no collective)",
                       "l2": "working set 4x134 MB per step > 126 MB L2 (no flush needed)",
                       "bytes_per_step_per_gpu": bytes_step},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": {"value": round(e2e_val, 3), "unit": UNIT, "h2d_bytes_per_step": numel * esz,
                    "d2h_bytes_per_step": numel * esz, "steps": e_steps,
                    "ms_per_step": round(e_ms / e_steps, 4),
                    "path": "pinned host -> paper_2110_01172_b200.dct_2d/idct_2d (torch CUDA) -> pinned host"},
            "gpu_launches": args.steps * (plan.stage_count(_sdct.DCT_2D) + plan.stage_count(_sdct.IDCT_2D)),
            "clocks": clk,
            "cufft": cufft,
            "parity": {"round_trip_rel_l2": rt_err, "e2e_round_trip_rel_l2": e2e_err},
        }
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--size", type=int, default=4096)
    ap.add_argument("--dtype", choices=["float64", "float32"], default="float64")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--cpu-budget", type=float, default=12.0, help="seconds of CPU baseline sampling")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
