"""bench.py's N>1 path (one process per rank, views sharded round-robin,
barrier + max-over-ranks timing) launched the way the driver launches it.
On a 1-GPU box both ranks share cuda:0 over gloo (BS_BENCH_SHARED_GPU=1,
test-only); on the 8-GPU node the same code runs one rank per GPU on NCCL."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("impl", ["b200", "reference"])
def test_bench_two_ranks(impl):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    args = ["--steps", "20", "--warmup", "3", "--no-extras"] if impl == "b200" else \
        ["--impl", "reference", "--steps", "1", "--warmup", "0"]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29561" if impl == "b200" else "29562",
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
    else:
        assert d["scaling"] == "weak" and d["gpu_launches"] > 0
