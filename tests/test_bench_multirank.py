"""bench.py's N>1 path (one process per rank; the default SURVEY 8e batch
mode: every step is the fixed batch of 64 orbit views split contiguously over
the ranks with sharding.batch_view_ids; --batch 0: one view per rank per
step; barrier + max-over-ranks timing) launched the way the driver launches it.
On a 1-GPU box both ranks share cuda:0 over gloo (BS_BENCH_SHARED_GPU=1,
test-only); on the 8-GPU node the same code runs one rank per GPU on NCCL."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("impl", ["b200", "b200_weak", "reference"])
def test_bench_two_ranks(impl):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    args = {"b200": ["--steps", "3", "--warmup", "3", "--no-extras"],
            "b200_weak": ["--steps", "20", "--warmup", "3", "--no-extras", "--batch", "0"],
            "reference": ["--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "0"]}[impl]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", {"b200": "29561", "b200_weak": "29563", "reference": "29562"}[impl],
           "bench.py", "--gpus", "2"] + args
    env = dict(os.environ, BS_BENCH_SHARED_GPU="1", BS_CLOCKS="off")
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0
    if impl == "reference":
        assert d["impl"] == "reference"
    elif impl == "b200":  # 3 steps x the 64-view batch, 32 views per rank
        assert d["scaling"] == "strong" and d["views_per_step"] == 64 and d["gpu_launches"] > 0
    else:
        assert d["scaling"] == "weak" and d["views_per_step"] == 2 and d["gpu_launches"] > 0
