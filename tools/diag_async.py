"""Host-side cost of one FramePipeline.forward in async vs sync mode (diagnostic)."""
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
for mode in (True, False, True, False):
    fp = api.FramePipeline(W, H, 16, 16, "cuda", 0, async_mode=mode)
    for i in range(10):
        fp.forward(d, n, cams[i % 64])
    fp.sync()
    torch.cuda.synchronize()
    host = []
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(100)]
    t_all = time.perf_counter()
    for i in range(100):
        ev[i][0].record()
        t0 = time.perf_counter()
        fp.forward(d, n, cams[i % 64])
        host.append(time.perf_counter() - t0)
        ev[i][1].record()
    fp.sync()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t_all
    gpu = [a.elapsed_time(b) for a, b in ev]
    print(f"async={mode}: host call p50 {np.median(host)*1e3:.3f} ms max {max(host)*1e3:.3f}; "
          f"gpu step p50 {np.median(gpu):.3f} ms; wall/frame {wall*10:.3f} ms")
    fp.close()
