#!/usr/bin/env python
"""Benchmark of the hot path (BASELINE.json metric: 2D DCT/IDCT ms and
effective GB/s vs the HBM roofline, with the reference CPU path alongside).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c2|c1|c3|c4|c5] [--dtype float64|float32]

Default workload c2 = BASELINE configs[1], the configuration the headline is
quoted on: one step = dct_2d then idct_2d of one 4096x4096 fp64 image. The
other BASELINE configs are selectable (c1 1024^2 fp64 DCT, c3 2048^2 IDXST/IDCT
composites, c4 256^3 fp32 3D DCT, c5 batched 512 x 2048^2 fp32 DCT sharded
over the ranks).

Algorithmic bytes per transform = 2 * numel * sizeof(T) (read the input once,
write the output once). `value` = those bytes for all ranks /
max-over-ranks device time, inputs resident in HBM. Workloads whose working
set fits in the 126 MB L2 rotate over enough input/output sets that no step
re-reads L2-resident data (said in config.l2).

N > 1 (torchrun): c1-c4 = every rank transforms its own images (independent
objects, no data-path collective, weak scaling); c5 = the fixed 512-image
batch is split into contiguous shards (strong scaling). Rank 0 prints one JSON
line.

--impl reference: the unmodified reference CPU library (oracle/_ref, built from
/root/reference by oracle/Makefile; the C restatement when absent) on this
host's cores, same workload, metric and unit (fp64: the reference is fp64-only).
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
# Workloads (BASELINE.json configs). mode "chain": kinds applied in sequence
# to the step's input; "fan": each kind applied to the same input; "force":
# the spectral force-field step (dct_2d, weighting, both composites), whose
# `kinds` list the transforms it is made of.
WORKLOADS = {
    "c2": dict(dims=(4096, 4096), kinds=["dct_2d", "idct_2d"], mode="chain", dtype="float64", batch=1,
               desc="2D DCT-II -> IDCT round trip 4096x4096 {dt} per rank (BASELINE configs[1])"),
    "c1": dict(dims=(1024, 1024), kinds=["dct_2d"], mode="chain", dtype="float64", batch=1,
               desc="2D DCT-II 1024x1024 {dt} per rank (BASELINE configs[0])"),
    "c3": dict(dims=(2048, 2048), kinds=["dct_2d", "idct_idxst_2d", "idxst_idct_2d"], mode="force",
               dtype="float64", batch=1,
               desc="DREAMPlace-style field step 2048x2048 {dt} per rank: dct_2d, weighting, IDCT/IDXST + "
                    "IDXST/IDCT composites (BASELINE configs[2]; force_demo_fields)"),
    "c4": dict(dims=(256, 256, 256), kinds=["dct_3d"], mode="chain", dtype="float32", batch=1,
               desc="3D DCT-II 256^3 {dt} per rank (BASELINE configs[3])"),
    "c5": dict(dims=(2048, 2048), kinds=["dct_2d"], mode="chain", dtype="float32", batch=512, sharded=True,
               desc="batched DCT-II 512 x 2048x2048 {dt}, batch sharded over ranks (BASELINE configs[4])"),
    # SURVEY §8f next rows, measured like the configs
    "cz": dict(dims=(4096, 4096), kinds=["dct_2d", "idct_2d"], mode="compress", dtype="float64", batch=1,
               desc="compression round trip 4096x4096 {dt} per rank: dct_2d, |b| < median zeroed, "
                    "idct_2d * 4/(N1 N2) (compress.cpp:24-54 numeric core)"),
}
L2_BYTES = 126 * 1024 * 1024


def _numel(dims):
    n = 1
    for d in dims:
        n *= d
    return n


def _shard(w, world, rank):
    """Contiguous batch shard of this rank (c5) or the per-rank batch."""
    if not w.get("sharded"):
        return 0, w["batch"]
    from paper_2110_01172_b200.shard import shard_range

    lo, hi = shard_range(w["batch"], world, rank)
    return lo, hi - lo


# ---------------------------------------------------------------------------
def cpu_reference_rate(w, budget_s: float, max_steps: int | None = None):
    """The reference CPU path (oracle/_ref, all host threads; the C
    restatement when the reference is not built) on a bounded sample of the
    workload: whole steps, or for batched c5 a few images. Returns (GB/s of
    the workload's algorithmic bytes, seconds per sampled unit, units timed,
    kind, sample description)."""
    import numpy as np

    import oracle

    dims, kinds = w["dims"], w["kinds"]
    x = np.random.default_rng(2).uniform(-1.0, 1.0, size=dims)
    if oracle.ref_available():
        kind = "reference"
        fns = [lambda a, k=k: oracle.ref.run(k, a, threads=0) for k in kinds]  # noqa: E731
        force = lambda a: oracle.ref.force_demo_fields(a, threads=0)  # noqa: E731
    else:
        kind = "port"
        fns = [getattr(oracle.port, k) for k in kinds]
        force = oracle.port.force_demo_fields

    def unit():
        if w["mode"] == "compress":
            import numpy as np_

            b = fns[0](x)
            fns[1](np_.where(np_.abs(b) < np_.median(np_.abs(b)), 0.0, b)) * (4.0 / b.size)
        elif w["mode"] == "force":
            force(x)
        elif w["mode"] == "chain":
            y = x
            for f in fns:
                y = f(y)
        else:
            for f in fns:
                f(x)

    t0 = time.perf_counter()
    unit()  # warm-up (also sizes the sample)
    t_u = time.perf_counter() - t0
    n = max(1, int(budget_s / max(t_u, 1e-3)))
    if max_steps is not None:
        n = min(n, max_steps)
    if kind == "reference" and w["mode"] in ("chain", "fan", "force"):
        # plans and input tensors built once outside the clock; only the
        # transform calls are timed (inside the reference library)
        if w["mode"] == "force":
            _, dt = oracle.ref.force_timed(x, threads=0, reps=n)
        else:
            dt, y = 0.0, x
            for k in kinds:
                out, s = oracle.ref.run_timed(k, y if w["mode"] == "chain" else x, threads=0, reps=n)
                dt += s
                y = out
        timing = "prebuilt plans, transform calls timed inside the library"
    else:
        t0 = time.perf_counter()
        for _ in range(n):
            unit()
        dt = (time.perf_counter() - t0) / n
        timing = "whole calls timed (plan built per call)" if kind == "reference" else "C restatement, 1 thread"
    bytes_unit = 2.0 * _numel(dims) * 8 * len(kinds)
    what = ("force_demo_fields" if w["mode"] == "force" else
            "dct_2d, threshold at the median |b|, idct_2d, 4/(N1 N2)" if w["mode"] == "compress" else
            " then ".join(kinds) if w["mode"] == "chain" else " + ".join(kinds))
    sample = (f"{n} x ({what}) of one {'x'.join(map(str, dims))} fp64 image on the host, {timing}, "
              f"threads=0 ({dt * 1e3:.1f} ms each)")
    if w.get("sharded"):
        sample += f"; the {w['batch']}-image batch is {w['batch']} such units (rate is per byte, batch-independent)"
    return bytes_unit / dt / 1e9, dt, n, kind, sample


# ---------------------------------------------------------------------------
def graph_time(fn, reps, stream, eager=False):
    """Average ms of fn() over `reps` back-to-back calls on `stream`, the calls
    captured once into a CUDA graph and replayed (so host launch latency, which
    exceeds the device time of the small configs, is not what gets timed).
    fn(sh) must launch on the raw stream handle sh. Falls back to eager launches
    (returned flag False) if capture fails or eager is requested."""
    import torch

    def eager_run():
        for _ in range(3):
            fn(stream.cuda_stream)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn(stream.cuda_stream)
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    if eager:
        return eager_run(), False
    try:
        g = capture_graph(lambda sh: [fn(sh) for _ in range(reps)], stream)
    except Exception:
        return eager_run(), False
    g.replay()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    g.replay()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, True


def graph_kernel_nodes(graph):
    """Kernel nodes of a captured torch CUDA graph (cudaGraphGetNodes +
    cudaGraphNodeGetType through the CUDA runtime), or None if unavailable."""
    import ctypes

    try:
        raw = graph.raw_cuda_graph()
        rt = None
        for name in ("libcudart.so.12", "libcudart.so"):
            try:
                rt = ctypes.CDLL(name)
                break
            except OSError:
                continue
        if rt is None:
            return None
        n = ctypes.c_size_t(0)
        if rt.cudaGraphGetNodes(ctypes.c_void_p(raw), None, ctypes.byref(n)) != 0:
            return None
        nodes = (ctypes.c_void_p * n.value)()
        if rt.cudaGraphGetNodes(ctypes.c_void_p(raw), nodes, ctypes.byref(n)) != 0:
            return None
        kinds = ctypes.c_int(0)
        count = 0
        for i in range(n.value):
            if rt.cudaGraphNodeGetType(ctypes.c_void_p(nodes[i]), ctypes.byref(kinds)) == 0 and kinds.value == 0:
                count += 1  # cudaGraphNodeTypeKernel
        return count
    except Exception:
        return None


def capture_graph(body, stream):
    """Capture body(sh) (launches on raw stream handle sh) into a CUDA graph."""
    import torch

    cs = torch.cuda.Stream(stream.device)
    cs.wait_stream(stream)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=cs, capture_error_mode="thread_local"):
        body(cs.cuda_stream)
    torch.cuda.synchronize()
    return g


def cufft_times(x, dims, batch, stream, reps, eager=False):
    """cuFFT R2C and C2R (D2Z / Z2D for fp64) of the same shape and batch,
    called directly through libcufft (ctypes; cufftPlanMany) so no framework
    copies or plan-cache effects are timed. Library baseline only (north_star:
    'cuFFT R2C on the same shape ... reported alongside'). Returns ms."""
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
    half = list(dims[:-1]) + [dims[-1] // 2 + 1]
    spec = torch.empty([batch] + half, dtype=torch.complex128 if f64 else torch.complex64, device=x.device)
    out = torch.empty_like(x)
    nn = (ctypes.c_int * len(dims))(*dims)
    pf, pi = ctypes.c_int(0), ctypes.c_int(0)
    for pl, ty in ((pf, fwd_type), (pi, inv_type)):
        rc = lib.cufftPlanMany(ctypes.byref(pl), len(dims), nn, None, 1, 0, None, 1, 0, ty, batch)
        if rc != 0:
            raise RuntimeError(f"cufftPlanMany failed ({rc})")
        lib.cufftSetStream(pl, ctypes.c_void_p(stream.cuda_stream))
    exf = lib.cufftExecD2Z if f64 else lib.cufftExecR2C
    exi = lib.cufftExecZ2D if f64 else lib.cufftExecC2R
    xi, so, oo = ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(spec.data_ptr()), ctypes.c_void_p(out.data_ptr())
    res = []
    for ex, pl, a_, b_ in ((exf, pf, xi, so), (exi, pi, so, oo)):
        for _ in range(3):
            if ex(pl, a_, b_) != 0:
                raise RuntimeError("cufftExec failed")

        def call(sh, ex=ex, pl=pl, a_=a_, b_=b_):
            lib.cufftSetStream(pl, ctypes.c_void_p(sh))
            ex(pl, a_, b_)

        res.append(graph_time(call, reps, stream, eager)[0])
        lib.cufftSetStream(pl, ctypes.c_void_p(stream.cuda_stream))
    lib.cufftDestroy(pf)
    lib.cufftDestroy(pi)
    return res[0], res[1]


# ---------------------------------------------------------------------------
def job_config(args, w, world: int) -> dict:
    """The workload description both arms print (identical dicts)."""
    dtype = args.dtype or w["dtype"]
    return {"workload": w["desc"].format(dt=dtype), "name": args.workload,
            "global_batch": w["batch"] if w.get("sharded") else world * w["batch"],
            "parallelism": (f"batch sharded x{world} (contiguous shards, no collective)" if w.get("sharded")
                            else f"replicas x{world} (independent images, no collective)")}


def run_reference(args, rank: int, world: int):
    if rank != 0:
        return
    w = WORKLOADS[args.workload]
    # bound the whole --steps K --warmup W run to a few minutes of CPU time
    rate, dt, steps, kind, sample = cpu_reference_rate(w, budget_s=150.0, max_steps=args.steps)
    cores, quota = _cores()
    line = {
        "impl": "reference", "metric": METRIC, "value": round(rate, 4), "unit": UNIT,
        "n_gpus": world, "steps": steps, "warmup": args.requested_warmup, "ms_per_step": round(dt * 1e3, 3),
        "higher_is_better": True, "scaling": "strong" if w.get("sharded") else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic uniform(-1,1)",
        "config": job_config(args, w, world),
        "measurement": {"requested_steps": args.steps, "requested_warmup": args.requested_warmup,
                        "note": "reference is fp64-only; CPU arm runs on rank 0 (host cores), one warm-up unit"},
        "cpu_baseline": {"value": round(rate, 4), "unit": UNIT, "cores": cores, "kind": kind,
                         "cgroup_cpu_quota": quota, "sample": sample},
        "e2e": {"value": round(rate, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def run_ours(args, rank: int, world: int, local_rank: int, backend: str | None = None):
    import torch
    import torch.distributed as dist

    import paper_2110_01172_b200 as sd
    from paper_2110_01172_b200 import _sdct

    w = WORKLOADS[args.workload]
    dtype = args.dtype or w["dtype"]
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dims = tuple(w["dims"])
    dt = torch.float64 if dtype == "float64" else torch.float32
    esz = 8 if dt == torch.float64 else 4
    lo, B = _shard(w, world, rank)
    numel = _numel(dims)
    item_bytes = numel * esz
    kinds = [getattr(_sdct, k.upper()) for k in w["kinds"]]
    bytes_transform = 2.0 * numel * esz * B  # one kind over this rank's batch
    bytes_step = bytes_transform * len(kinds)  # this rank
    # whole-job bytes per step: every rank's own images, or the one sharded batch
    job_bytes_step = world * bytes_step if not w.get("sharded") else 2.0 * numel * esz * w["batch"] * len(kinds)

    # rotation sets so that no step reads L2-resident inputs of the previous one
    set_bytes = item_bytes * B * (2 if w["mode"] == "fan" else 3 if w["mode"] == "force" else len(kinds) + 1)
    rot = 1 if set_bytes >= 2 * L2_BYTES else -(-2 * L2_BYTES // set_bytes) + 1
    g = torch.Generator(device="cpu").manual_seed(2 + rank)
    x_host = (torch.rand((B,) + dims, generator=g, dtype=torch.float64) * 2 - 1).to(dt) if B <= 4 else None
    xs = []
    for r in range(rot):
        if x_host is not None:
            xs.append((x_host if r == 0 else torch.roll(x_host, r, dims=-1)).to(dev))
        else:  # large batches: generate on the device (no multi-GB host copy)
            gd = torch.Generator(device=dev).manual_seed(5 + rank + 1000 * r)
            xs.append((torch.rand((B,) + dims, generator=gd, dtype=torch.float64, device=dev) * 2 - 1).to(dt))
    nbuf = len(kinds) if w["mode"] == "chain" else len(kinds)
    outs = [[torch.empty_like(xs[0]) for _ in range(nbuf)] for _ in range(rot)]
    stream = torch.cuda.current_stream(dev)
    s = stream.cuda_stream
    plan = sd.plan_for(dims, B, dtype, local_rank)
    ws = torch.empty(plan.workspace_bytes, dtype=torch.uint8, device=dev)

    eps_c = 0.0
    zeroed = torch.zeros(1, dtype=torch.int64, device=dev)
    if w["mode"] == "compress":
        # threshold = the median coefficient magnitude of the (first) input
        b0 = torch.empty_like(xs[0])
        plan.run(_sdct.DCT_2D, xs[0].data_ptr(), b0.data_ptr(), s, ws.data_ptr())
        eps_c = float(b0.abs().median().item())
        del b0

    def step(i, sh=None):
        sh = s if sh is None else sh
        r = i % rot
        src = xs[r]
        if w["mode"] == "force":
            plan.force_fields(src.data_ptr(), outs[r][0].data_ptr(), outs[r][1].data_ptr(), sh, ws.data_ptr())
            return
        if w["mode"] == "compress":
            plan.compress(src.data_ptr(), outs[r][0].data_ptr(), eps_c, zeroed.data_ptr(), sh, ws.data_ptr())
            return
        for j, k in enumerate(kinds):
            dst = outs[r][j]
            plan.run(k, src.data_ptr(), dst.data_ptr(), sh, ws.data_ptr())
            if w["mode"] == "chain":
                src = dst

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # parity spot check of this rank's own data
    step(0)
    torch.cuda.synchronize()
    parity = {}
    if w["mode"] == "chain" and w["kinds"] == ["dct_2d", "idct_2d"]:
        scale = numel / 4.0
        parity["round_trip_rel_l2"] = float(((outs[0][1] / scale - xs[0]).norm() / xs[0].norm()).item())
        if rank == 0:
            # the forward transform of the timed loop's input against the C
            # oracle (oracle/sdct_oracle.c, a few s at 4096^2 on one host core)
            import oracle

            x0 = xs[0][0].double().cpu().numpy()
            parity["dct_2d_rel_l2_vs_oracle"] = float(
                oracle.rel_l2(outs[0][0][0].double().cpu().numpy(), oracle.port.dct_2d(x0)))
    elif w["mode"] == "compress":
        zeroed.zero_()
        step(0)
        torch.cuda.synchronize()
        parity["zeroed_fraction"] = float(zeroed.item()) / (B * numel)
    elif rank == 0 and w["mode"] == "force":
        import oracle

        w1, w2 = oracle.port.force_demo_fields(xs[0][0].double().cpu().numpy())
        parity["xi1_rel_l2_vs_oracle"] = float(oracle.rel_l2(outs[0][0][0].double().cpu().numpy(), w1))
        parity["xi2_rel_l2_vs_oracle"] = float(oracle.rel_l2(outs[0][1][0].double().cpu().numpy(), w2))
    elif w.get("sharded"):
        # every rank checks the first and last image of its own shard against
        # the C oracle (the shard-boundary images of BASELINE.md §4); the line
        # reports the worst over ranks
        import oracle

        errs = []
        for bi in sorted({0, B - 1}):
            x0 = xs[0][bi].double().cpu().numpy()
            errs.append(oracle.rel_l2(outs[0][0][bi].double().cpu().numpy(), oracle.port.dct_2d(x0)))
        parity["shard_images_checked"] = [lo, lo + B - 1]
        parity["dct_2d_rel_l2_vs_oracle_max_over_ranks"] = max_over_ranks(max(errs))
        parity["images_checked_total"] = len({0, B - 1}) * world
    elif rank == 0:
        import oracle

        for j, k in enumerate(w["kinds"]):
            if w["mode"] == "chain" and j > 0:
                break
            x0 = xs[0][0].double().cpu().numpy()
            ref = getattr(oracle.port, k)(x0) if numel <= 1 << 22 else None
            if ref is not None:
                parity[f"{k}_rel_l2_vs_oracle"] = float(oracle.rel_l2(outs[0][j][0].double().cpu().numpy(), ref))

    # the K timed steps are captured once into a CUDA graph (the same plan.run
    # launches, programmatic dependent launch edges kept) and replayed: the
    # small configs' kernels run shorter than Python + driver launch latency,
    # so eager launching would time the host, not the device
    graph, graph_note = None, "eager launches (--eager)"
    if not args.eager:
        try:
            graph = capture_graph(lambda sh: [step(j, sh) for j in range(args.steps)], stream)
            graph_note = f"CUDA graph of the {args.steps} steps, replayed (captured once before warm-up)"
        except Exception as e:  # pragma: no cover - reported, falls back to eager
            graph_note = f"eager launches (graph capture failed: {str(e)[:120]})"

    # kernels launched inside the timed region: the kernel nodes of the captured
    # graph (the plan's own launches only: the step calls nothing else), else the
    # plan's stage count per step (force fields on a single-image fast plan: the
    # two composites run as one paired row launch and one paired column launch)
    n_launch = None
    if graph is not None:
        n_launch = graph_kernel_nodes(graph)
    if n_launch is None:
        per_step = sum(plan.stage_count(k) for k in kinds)
        if w["mode"] == "force" and B == 1 and plan.fast:
            per_step = plan.stage_count(kinds[0]) + 2
        n_launch = args.steps * per_step

    clocks = ClockSampler(local_rank)
    clocks.start()
    t_w = time.perf_counter()
    i = 0
    while i < args.warmup or time.perf_counter() - t_w < 1.0:  # >= W steps and >= 1 s soak
        if graph is not None:
            graph.replay()
            i += args.steps
            torch.cuda.synchronize()
            continue
        step(i)
        i += 1
        if i % 20 == 0:
            torch.cuda.synchronize()
    warm_done = i
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    if graph is not None:
        graph.replay()
    else:
        for j in range(args.steps):
            step(j)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms = e0.elapsed_time(e1)
    clk = clocks.stop()
    ms = max_over_ranks(ms)
    ms_per_step = ms / args.steps
    value = job_bytes_step * args.steps / (ms / 1e3) / 1e9

    # ---- per-kernel timing (roofline of the dominant kernel) ----------------
    # graph mode: for each kernel of the step, n_inst back-to-back launches of
    # that kernel alone on the timed loop's rotating buffers (inputs cold as in
    # the step; the workspace intermediate as its producer leaves it), captured
    # into a CUDA graph and timed with events around the replay. Eager mode:
    # the timed loop's steps again with an event between every kernel launch.
    peak, peak_kind = _peaks()
    stage_list = [(kn, k, st) for kn, k in zip(w["kinds"], kinds) for st in range(plan.stage_count(k))]
    n_inst = max(10, min(args.steps, 50))
    torch.cuda.synchronize()
    kernels = []
    kt_graph = graph is not None
    if kt_graph:
        for ki, (kn, k) in enumerate(zip(w["kinds"], kinds)):
            for st in range(plan.stage_count(k)):
                def one(sh, j=[0], ki=ki, k=k, st=st):
                    r = j[0] % rot
                    j[0] += 1
                    src = outs[r][ki - 1] if (w["mode"] == "chain" and ki > 0) else xs[r]
                    plan.run_stage(k, st, src.data_ptr(), outs[r][ki].data_ptr(), sh, ws.data_ptr())

                avg, ok = graph_time(one, n_inst, stream)
                kt_graph = kt_graph and ok
                kernels.append({"kernel": f"{kn}.stage{st}", "ms": avg, "gbs": bytes_transform / (avg / 1e3) / 1e9})
    else:
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(len(stage_list) + 1)] for _ in range(n_inst)]
        for j in range(n_inst):
            r = j % rot
            src = xs[r]
            evs[j][0].record(stream)
            e_i = 1
            for kn, k in zip(w["kinds"], kinds):
                dst = outs[r][w["kinds"].index(kn)]
                for st in range(plan.stage_count(k)):
                    plan.run_stage(k, st, src.data_ptr(), dst.data_ptr(), s, ws.data_ptr())
                    evs[j][e_i].record(stream)
                    e_i += 1
                if w["mode"] == "chain":
                    src = dst
        torch.cuda.synchronize()
        for i, (kn, k, st) in enumerate(stage_list):
            ts = [evs[j][i].elapsed_time(evs[j][i + 1]) for j in range(n_inst)]
            avg = sum(ts) / len(ts)
            kernels.append({"kernel": f"{kn}.stage{st}", "ms": avg, "gbs": bytes_transform / (avg / 1e3) / 1e9})
    # cold: each kernel alone after an L2 flush (ncu-like conditions), for reference
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    cold = []
    src = xs[0]
    for kn, k in zip(w["kinds"], kinds):
        dst = outs[0][0]
        for st in range(plan.stage_count(k)):
            times = []
            for _ in range(6):
                flush.fill_(1)  # evict L2 (256 MB > 126 MB) outside the timed launch
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                plan.run_stage(k, st, src.data_ptr(), dst.data_ptr(), s, ws.data_ptr())
                b.record(stream)
                torch.cuda.synchronize()
                times.append(a.elapsed_time(b))
            avg = sum(times[2:]) / len(times[2:])
            cold.append({"kernel": f"{kn}.stage{st}", "ms": round(avg, 4),
                         "gbs": round(bytes_transform / (avg / 1e3) / 1e9, 2)})
        plan.run(k, src.data_ptr(), dst.data_ptr(), s, ws.data_ptr())  # dst valid for the next kind
        if w["mode"] == "chain":
            src = dst.clone()
    torch.cuda.synchronize()
    dom = max(kernels, key=lambda k_: k_["ms"])
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            traffic = json.load(f).get(f"{args.workload}:{dtype}:{dom['kernel']}")
    except Exception:
        pass
    roofline = {"bound": "hbm", "achieved": round(dom["gbs"], 2), "peak": peak, "unit": "GB/s",
                "frac": round(dom["gbs"] / peak, 4), "traffic": traffic, "kernel": dom["kernel"],
                "peak_kind": peak_kind, "per_launch_bytes": bytes_transform,
                "timing": (f"live, CUDA graph: {n_inst} back-to-back launches of each kernel alone on the timed "
                           "loop's rotating buffers, events around the graph replay (programmatic dependent launch "
                           "overlaps each launch's prologue with its predecessor's tail, as in the step)"
                           if kt_graph else
                           f"live: {n_inst} steps of the timed loop with an event between kernels (the events "
                           "stop programmatic dependent launch from overlapping kernel tails, so the per-kernel "
                           "times sum to more than ms_per_step)"),
                "all_kernels": [{k2: (round(v, 4) if isinstance(v, float) else v) for k2, v in k_.items()}
                                for k_ in kernels],
                "cold_l2_flushed": cold,
                "step_frac": round(value / world / peak, 4),
                **({"note": ("force step: on this single-image fast plan the two composites run as ONE paired row "
                             "launch and ONE paired column launch with the field weighting in the row loads "
                             "(gpu_launches counts those); the per-kernel entries time each composite's two "
                             "kernels unpaired and unweighted through the stage API")}
                   if w["mode"] == "force" else {}),
                "step_frac_2pass_normalised": round(2 * value / world / peak, 4)}

    # ---- cuFFT on the same shape (library baseline, reported alongside) -----
    cufft = {}
    try:
        reps = 10 if B > 1 else 20
        # both sides timed the same way: reps calls on one input, captured
        # into a CUDA graph and replayed (eager with --eager)
        r2c, c2r = cufft_times(xs[0], list(dims), B, stream, reps, args.eager)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        ours = {}
        src = xs[0]
        for kn, k in zip(w["kinds"], kinds):
            ours[kn] = graph_time(lambda sh, k=k: plan.run(k, src.data_ptr(), outs[0][0].data_ptr(), sh,
                                                          ws.data_ptr()), reps, stream, args.eager)[0]
        cufft = {"api": "libcufft cufftPlanMany + cufftExec{D2Z,Z2D|R2C,C2R}, plan built outside timing",
                 "timing": "eager launches" if args.eager else "CUDA graph replay of the repeated calls (both sides)",
                 "r2c_ms": round(r2c, 4), "c2r_ms": round(c2r, 4)}
        if len(dims) == 2 and "dct_2d" in w["kinds"]:
            # row-column DCT on the same shape (north_star: "reported alongside"):
            # dct_2d_rowcol runs one pass per axis (gather, FFT along each axis,
            # postprocess) on the generic GPU path
            k_rc = _sdct.DCT_2D_ROWCOL
            plan.run(k_rc, xs[0].data_ptr(), outs[0][0].data_ptr(), s, 0)
            torch.cuda.synchronize()
            rc_ms = graph_time(lambda sh: plan.run(k_rc, xs[0].data_ptr(), outs[0][0].data_ptr(), sh, 0), 3,
                               stream, args.eager)[0]
            cufft["rowcol_dct_2d_ms"] = round(rc_ms, 4)
        for kn, v in ours.items():
            cufft[f"{kn}_ms"] = round(v, 4)
            base = r2c if kn.startswith("dct") else c2r
            cufft[f"{kn}_over_{'r2c' if kn.startswith('dct') else 'c2r'}"] = round(v / base, 3)
    except Exception as e:  # pragma: no cover - reported, not fatal
        cufft = {"error": str(e)}

    # ---- end to end through the public API with host buffers ---------------
    # sd.stream_host: per step, every item of the step goes pinned host -> H2D
    # -> the workload's transforms -> D2H -> pinned host; consecutive items
    # are software-pipelined over three streams (copies overlap the kernels
    # and each other: PCIe is full duplex). Timed with CUDA events on the
    # caller's stream, which the pipeline forks from and joins back into.
    x_pin = xs[0][:1].cpu().pin_memory()
    out_pin = torch.empty_like(x_pin).pin_memory()
    chains = ([w["kinds"]] if w["mode"] == "chain" else [[k] for k in w["kinds"]] if w["mode"] == "fan" else [])
    if w["mode"] == "compress":
        chains = []
    e_steps = 1 if B > 16 else max(5, min(args.steps, 50))
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    if w["mode"] == "compress":
        # sd.compress on a device tensor: image in, reconstruction out every step
        xd = torch.empty_like(xs[0][:1])

        def e2e_compress():
            xd.copy_(x_pin, non_blocking=True)
            rec, _ = sd.compress(xd[0], eps_c)
            out_pin[0].copy_(rec, non_blocking=True)

        e2e_compress()
        torch.cuda.synchronize()
        barrier()
        a.record(stream)
        for _ in range(e_steps):
            e2e_compress()
        b.record(stream)
        n_out = 1
    elif w["mode"] == "force":
        # sd.force_demo_fields on a device tensor, with the density copied in and
        # both fields copied out every step; consecutive steps round-robin over
        # three streams (each call has its own coefficient scratch), so one
        # step's D2H overlaps the next one's H2D and kernels (PCIe is full duplex)
        lanes = 3
        lstreams = [torch.cuda.Stream(dev) for _ in range(lanes)]
        xdl = [torch.empty_like(xs[0][:1]) for _ in range(lanes)]
        o1l = [torch.empty_like(out_pin).pin_memory() for _ in range(lanes)]
        o2l = [torch.empty_like(out_pin).pin_memory() for _ in range(lanes)]

        def e2e_force(i):
            k = i % lanes
            with torch.cuda.stream(lstreams[k]):
                xdl[k].copy_(x_pin, non_blocking=True)
                f1, f2 = sd.force_demo_fields(xdl[k][0])
                o1l[k][0].copy_(f1, non_blocking=True)
                o2l[k][0].copy_(f2, non_blocking=True)

        for i in range(lanes):
            e2e_force(i)
        torch.cuda.synchronize()
        barrier()
        a.record(stream)
        for ls_ in lstreams:
            ls_.wait_stream(stream)
        for i in range(e_steps):
            e2e_force(i)
        for ls_ in lstreams:
            stream.wait_stream(ls_)
        b.record(stream)
        out_pin.copy_(o1l[(e_steps - 1) % lanes])
        n_out = 2
    else:
        for ch in chains:
            sd.stream_host(ch, x_pin, out_pin, count=3, device=local_rank)  # warm-up (lane buffers)
        torch.cuda.synchronize()
        barrier()
        a.record(stream)
        for ch in chains:
            sd.stream_host(ch, x_pin, out_pin, count=e_steps * B, device=local_rank, sync=False)
        b.record(stream)
        n_out = len(chains)
    torch.cuda.synchronize()
    e_ms = max_over_ranks(a.elapsed_time(b))
    e2e_val = job_bytes_step * e_steps / (e_ms / 1e3) / 1e9
    if w["mode"] == "chain" and w["kinds"] == ["dct_2d", "idct_2d"]:
        x0 = x_pin[0].to(torch.float64)
        parity["e2e_round_trip_rel_l2"] = float(((out_pin[0].to(torch.float64) / (numel / 4.0) - x0).norm()
                                                 / x0.norm()).item())

    # ---- second e2e figure: the reference's own Python surface on numpy -------
    # sdct.dct_2d(numpy) -> sdct.idct_2d(numpy): float64 pageable host arrays in
    # and out of every call (as the reference module takes and returns them),
    # device plans from the C++ plan cache. Host-synchronous, so wall clock.
    e2e_np = None
    if (w["mode"] == "chain" and w["kinds"] == ["dct_2d", "idct_2d"] and dtype == "float64" and B == 1):
        import numpy as np

        x_np = xs[0][0].double().cpu().numpy()
        y_np = sd.idct_2d(sd.dct_2d(x_np))  # warm: plan cache + allocator
        n_np = 5
        barrier()
        t_np = time.perf_counter()
        for _ in range(n_np):
            y_np = sd.idct_2d(sd.dct_2d(x_np))
        np_ms = (time.perf_counter() - t_np) * 1e3 / n_np
        np_ms = max_over_ranks(np_ms)
        e2e_np = {"value": round(bytes_step / (np_ms / 1e3) / 1e9, 3), "unit": UNIT, "ms_per_step": round(np_ms, 4),
                  "h2d_bytes_per_step": 2 * x_np.nbytes, "d2h_bytes_per_step": 2 * x_np.nbytes,
                  "path": "sdct.dct_2d(numpy) -> sdct.idct_2d(numpy): reference Python surface, float64 pageable "
                          "host arrays per call, cached device plans, wall clock",
                  "round_trip_rel_l2": float(np.linalg.norm(y_np / (numel / 4.0) - x_np) / np.linalg.norm(x_np))}

    # ---- CPU baseline (rank 0, N = 1 only) -----------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        rate, dtr, n_units, kind, sample = cpu_reference_rate(w, budget_s=args.cpu_budget)
        cores, quota = _cores()
        cpu = {"value": round(rate, 4), "unit": UNIT, "cores": cores if kind == "reference" else 1, "kind": kind,
               "cgroup_cpu_quota": quota, "sample": sample}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.requested_warmup, "ms_per_step": round(ms_per_step, 5),
            "higher_is_better": True, "scaling": "strong" if w.get("sharded") else "weak", "vs_baseline": None,
            "dtype": "f64" if dt == torch.float64 else "f32",
            "data": "synthetic uniform(-1,1), device-resident",
            "config": job_config(args, w, world),
            "measurement": {"launch": graph_note, "l2": ("working set per step > 2x the 126 MB L2 (no flush needed)" if rot == 1 else
                                   f"inputs/outputs rotate over {rot} sets ({rot * set_bytes / 2**20:.0f} MB > 2x L2)"),
                            "bytes_per_step_per_gpu": bytes_step, "warmup_steps_run": warm_done,
                            "warmup_rule": f">= {args.warmup} untimed steps and >= 1 s of soak before timing",
                            "ranks": world, "control_plane": backend or "none (1 rank)",
                            "devices": torch.cuda.device_count()},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": {"value": round(e2e_val, 3), "unit": UNIT,
                    "h2d_bytes_per_step": item_bytes * B * max(1, len(chains)),
                    "d2h_bytes_per_step": item_bytes * B * n_out, "steps": e_steps,
                    "ms_per_step": round(e_ms / e_steps, 4),
                    "path": ("pinned host -> paper_2110_01172_b200.force_demo_fields (torch CUDA; steps "
                             "round-robin over 3 streams) -> pinned host"
                             if w["mode"] == "force" else
                             "pinned host -> paper_2110_01172_b200.compress (torch CUDA) -> pinned host"
                             if w["mode"] == "compress" else
                             f"pinned host -> paper_2110_01172_b200.stream_host({w['kinds']}) "
                             "(sdct_exec_host_pipelined, 3 overlapped lanes) -> pinned host")},
            "e2e_numpy": e2e_np,
            "gpu_launches": n_launch,
            "clocks": clk,
            "cufft": cufft,
            "parity": parity,
        }
        print(json.dumps(line), flush=True)


def _free_port() -> int:
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def spawn_ranks(n: int) -> int:
    """`python bench.py --gpus N` without torchrun: re-launch this script as N
    ranks (one process per GPU, the torchrun environment contract) on
    127.0.0.1 and wait for all of them. Rank 0 prints the JSON line."""
    port = _free_port()
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n), LOCAL_WORLD_SIZE=str(n),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + sys.argv[1:], env=env))
    rc = 0
    for p in procs:
        rc = max(rc, p.wait())
    return rc


def dry_orchestration(args, rank: int, world: int):
    """The multi-rank control plane of run_ours without the GPU work: gloo
    process group, this rank's shard, barrier, max-over-ranks of a per-rank
    'time', rank 0 prints one JSON line (tests/test_dist.py)."""
    import torch
    import torch.distributed as dist

    w = WORKLOADS[args.workload]
    if world > 1:
        dist.init_process_group("gloo")
    lo, b = _shard(w, world, rank)
    t = torch.tensor([10.0 + rank, float(lo), float(lo + b)], dtype=torch.float64)
    if world > 1:
        dist.barrier()
        got = [torch.zeros(3, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(got, t)
        dist.destroy_process_group()
    else:
        got = [t]
    if rank == 0:
        print(json.dumps({"n_gpus": world, "config": job_config(args, w, world),
                          "ms_max_over_ranks": max(float(g[0]) for g in got),
                          "shards": [[int(g[1]), int(g[2])] for g in got]}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c2")
    ap.add_argument("--dtype", choices=["float64", "float32"], default=None,
                    help="override the workload's dtype (c2 runs fp64 by default)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--eager", action="store_true", help="launch the timed steps eagerly (no CUDA graph)")
    ap.add_argument("--cpu-budget", type=float, default=12.0, help="seconds of CPU baseline sampling")
    ap.add_argument("--dry-orchestration", action="store_true",
                    help="test hook: rank launch, shards and the max-over-ranks reduction only (gloo, no GPU)")
    args = ap.parse_args()
    args.requested_warmup = args.warmup
    if args.warmup < 3:
        args.warmup = 3
    launched = "WORLD_SIZE" in os.environ
    if args.impl == "reference":
        # the reference CPU arm runs on rank 0 only (other torchrun ranks exit 0)
        world = int(os.environ.get("WORLD_SIZE", "1")) if launched else max(1, args.gpus)
        run_reference(args, int(os.environ.get("RANK", "0")), world)
        return
    if not launched and args.gpus > 1:
        sys.exit(spawn_ranks(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.dry_orchestration:
        dry_orchestration(args, rank, world)
        return
    backend = None
    if world > 1:
        import torch
        import torch.distributed as dist

        ndev = torch.cuda.device_count()
        dev_index = local_rank % ndev
        torch.cuda.set_device(dev_index)
        # one rank per GPU: NCCL carries the barrier and the max-over-ranks
        # timing reduction (there is no data-path collective). Ranks sharing a
        # device (a 1-GPU test box) use gloo: NCCL rejects duplicate GPUs.
        backend = "nccl" if ndev >= int(os.environ.get("LOCAL_WORLD_SIZE", world)) else "gloo"
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index))
        else:
            dist.init_process_group("gloo")
    else:
        dev_index = local_rank
    try:
        run_ours(args, rank, world, dev_index, backend)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
