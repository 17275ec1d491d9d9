"""Find slow steps in the bench-like loop: GPU event time vs host time per step (diagnostic)."""
import gc
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2412_17378_b200 import api  # noqa: E402

W, H, f, n = 1920, 1080, 1000.0, 1_000_000
cams = [api.camera(bench.orbit_view(k), (f, f), W, H) for k in range(64)]
g3d = api.gen_clustered_scene(n, cams[0])
d = api.g3d_to_device(g3d, "cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
mode = os.environ.get("MODE", "async") == "async"
fp = api.FramePipeline(W, H, 16, 16, "cuda", 0, async_mode=mode)
for i in range(10):
    fp.forward(d, n, cams[i % 64])
fp.sync()
torch.cuda.synchronize()
for rep in range(3):
    steps = 200
    st = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    en = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    host = []
    gc.disable()
    for i in range(steps):
        flush.zero_()
        st[i].record()
        t0 = time.perf_counter()
        fp.forward(d, n, cams[(10 + i) % 64])
        host.append((time.perf_counter() - t0) * 1e3)
        en[i].record()
    fp.sync()
    gc.enable()
    torch.cuda.synchronize()
    g = np.array([a.elapsed_time(b) for a, b in zip(st, en)])
    h = np.array(host)
    top = np.argsort(-g)[:4]
    print(f"rep {rep}: gpu mean {g.mean():.3f} p50 {np.median(g):.3f} max {g.max():.2f}; host p50 {np.median(h):.3f} "
          f"max {h.max():.2f}; slow steps " + ", ".join(f"#{i} gpu {g[i]:.2f} host {h[i]:.2f} host_next "
                                                      f"{h[min(i + 1, steps - 1)]:.2f}" for i in top))
