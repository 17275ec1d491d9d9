"""CPU: the N>1 path with world_size-2 gloo — view sharding covers every view
exactly once, ranks never share a view, and the timing reduction is a max."""
from __future__ import annotations

import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2412_17378_b200 import sharding


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    views = sharding.views_for_rank(rank, world, steps=32)
    mine = list(sharding.contiguous_shard(64, rank, world))
    batch = sharding.batch_view_ids(rank, world, steps=3)  # bench.py's default schedule
    t = sharding.max_over_ranks(10.0 + rank, dist, "cpu")
    import torch

    gathered = [torch.zeros(32, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(gathered, torch.tensor(views, dtype=torch.int64))
    gathered_c = [None] * world
    dist.all_gather_object(gathered_c, mine)
    gathered_b = [None] * world
    dist.all_gather_object(gathered_b, batch)
    if rank == 0:
        out.put((t, [g.tolist() for g in gathered], gathered_c, gathered_b))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharding_and_max():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    t, views, contig, batches = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert t == 11.0
    allv = views[0] + views[1]
    assert sorted(allv) == list(range(64))  # 2 ranks x 32 steps cover the orbit once
    assert set(contig[0]).isdisjoint(contig[1]) and sorted(contig[0] + contig[1]) == list(range(64))
    # batch mode: each of the 3 steps renders the 64-view batch exactly once over the ranks
    assert len(batches[0]) == len(batches[1]) == 3 * 32
    assert sorted(batches[0] + batches[1]) == sorted(list(range(64)) * 3)


def test_contiguous_shards_all_sizes():
    for world in (1, 2, 3, 4, 8):
        parts = [list(sharding.contiguous_shard(64, r, world)) for r in range(world)]
        assert sum(parts, []) == list(range(64))


def test_orbit_views_orthonormal():
    for k in (0, 31, 63):
        V = sharding.orbit_view(k)
        R = V[:3, :3].astype(np.float64)
        assert np.abs(R @ R.T - np.eye(3)).max() < 1e-5
        # pivot maps to itself
        assert np.allclose(V[:3, :3] @ [0, 0, 5.5] + V[:3, 3], [0, 0, 5.5], atol=1e-5)


def test_reference_arm_two_ranks_cpu():
    """bench.py --impl reference under torch.distributed.run with 2 ranks on
    CPU: rank 0 alone times the reference (C1, one complete frame) and
    prints one JSON line; rank 1 exits 0 without work."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2", "--impl", "reference",
           "--config", "c1", "--steps", "1", "--warmup", "1"]
    r = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["e2e"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
