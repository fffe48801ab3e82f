"""Multi-process host logic (gloo, world_size 2, CPU): batch shards are
disjoint, complete and balanced, and the timing reduction is max-over-ranks —
the same code paths bench.py uses under torchrun on NCCL."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2110_01172_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, total, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    s, e = shard.shard_range(total, world, rank)
    t = torch.tensor([s, e], dtype=torch.int64)
    out = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(out, t)
    ms = torch.tensor([10.0 + rank], dtype=torch.float64)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    if rank == 0:
        q.put(([tuple(o.tolist()) for o in out], float(ms.item())))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("total", [512, 7])
def test_gloo_world2_shards_cover_batch(total):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, total, q)) for r in range(world)]
    for p in procs:
        p.start()
    ranges, ms = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    covered = [i for s, e in ranges for i in range(s, e)]
    assert covered == list(range(total))
    sizes = [e - s for s, e in ranges]
    assert max(sizes) - min(sizes) <= 1
    assert ms == 11.0  # max over ranks


def test_shard_helpers():
    assert shard.shard_range(512, 8, 7) == (448, 512)
    assert shard.spot_check_indices(512, 4) == [0, 127, 128, 255, 256, 383, 384, 511]
    with pytest.raises(ValueError):
        shard.shard_range(10, 2, 2)


# ---- slab-decomposed 3D transform (paper_2110_01172_b200/slab3d.py) --------
def _slab_worker(rank, world, port, q):
    import numpy as np

    import oracle
    from paper_2110_01172_b200 import slab3d

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n1, n2, n3 = 8, 6, 5
    x = np.random.default_rng(3).uniform(-1, 1, (n1, n2, n3))
    s1 = n1 // world
    xl = torch.tensor(x[rank * s1:(rank + 1) * s1])
    # local transforms on CPU from the C restatement (the GPU kernels need a
    # device); the exchange logic under test is the same code the GPUs run
    wrap = lambda f: (lambda t: torch.tensor(f(t.numpy())))  # noqa: E731
    # the axis-0 leg: the 1D transform of every column of an (n1 x m) matrix
    ax0 = lambda f: (lambda t: torch.tensor(np.ascontiguousarray(f(np.ascontiguousarray(t.numpy().T)).T)))  # noqa: E731
    y = slab3d.dct_3d_slab(xl, n1, two_d=wrap(oracle.port.dct_2d), axis0=ax0(oracle.port.dct_direct_1d))
    z = slab3d.idct_3d_slab(y, n1, two_d=wrap(oracle.port.idct_2d), axis0=ax0(oracle.port.idct_direct_1d))
    ys = [torch.zeros_like(y) for _ in range(world)]
    zs = [torch.zeros_like(z) for _ in range(world)]
    dist.all_gather(ys, y)
    dist.all_gather(zs, z)
    if rank == 0:
        q.put((torch.cat(ys).numpy(), torch.cat(zs).numpy(), x))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_slab_3d_matches_full_transform():
    import oracle

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_slab_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    y, z, x = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert oracle.rel_l2(y, oracle.port.dct_3d(x)) <= 1e-13
    assert oracle.rel_l2(z / (x.size / 8), x) <= 1e-13


# ---- bench.py rank orchestration (what the driver's SCALE run exercises) ---
def _bench(*argv, env=None, timeout=240):
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    e = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "LOCAL_WORLD_SIZE")}
    e.update(env or {})
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), *argv], capture_output=True, text=True,
                       timeout=timeout, env=e)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


@pytest.mark.parametrize("gpus", [2, 4])
def test_bench_self_spawns_ranks(gpus):
    """`bench.py --gpus N` without torchrun launches N ranks itself (gloo
    control plane here), shards c5 contiguously and reduces max over ranks."""
    out = _bench("--dry-orchestration", "--gpus", str(gpus), "--workload", "c5")
    assert out["n_gpus"] == gpus
    assert out["ms_max_over_ranks"] == 10.0 + gpus - 1
    covered = [i for s, e in out["shards"] for i in range(s, e)]
    assert covered == list(range(512))


def test_bench_arms_print_identical_config():
    """Both arms describe the workload with the same config dict and n_gpus
    (the reference arm runs on rank 0 only)."""
    ours = _bench("--dry-orchestration", "--gpus", "2", "--workload", "c2")
    import oracle

    if not oracle.ref_available():
        pytest.skip("reference library not built")
    ref = _bench("--impl", "reference", "--gpus", "2", "--workload", "c1", "--steps", "1", "--warmup", "3")
    ours1 = _bench("--dry-orchestration", "--gpus", "2", "--workload", "c1")
    assert ref["config"] == ours1["config"]
    assert ref["n_gpus"] == ours1["n_gpus"] == ours["n_gpus"] == 2
    assert ref["impl"] == "reference" and ref["cpu_baseline"]["kind"] == "reference"
    assert "prebuilt plans" in ref["cpu_baseline"]["sample"]
