"""Bench-like loop (L2 flush between steps) in async vs sync frame mode with
per-stage events: where does the step time go (diagnostic)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2412_17378_b200 import _native as N  # noqa: E402
from paper_2412_17378_b200 import api  # noqa: E402

W, H, f, n = 1920, 1080, 1000.0, 1_000_000
cams = [api.camera(bench.orbit_view(k), (f, f), W, H) for k in range(64)]
g3d = api.gen_clustered_scene(n, cams[0])
d = api.g3d_to_device(g3d, "cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for mode in (True, False, True, False):
    fp = api.FramePipeline(W, H, 16, 16, "cuda", 0, async_mode=mode)
    for i in range(10):
        fp.forward(d, n, cams[i % 64])
    fp.sync()
    for flush_on in (True, False):
        N.call("bs_context_enable_timing", fp.ctx, 1)
        steps, stages = [], []
        for i in range(60):
            if flush_on:
                flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fp.forward(d, n, cams[(10 + i) % 64])
            b.record()
            fp.sync()
            torch.cuda.synchronize()
            steps.append(a.elapsed_time(b))
            stages.append(list(fp.stage_ms().values()))
        st = np.mean(stages, axis=0)
        print(f"async={mode} flush={flush_on}: step {np.median(steps):.3f} ms, stages {np.round(st, 3).tolist()} "
              f"sum {st.sum():.3f}")
        N.call("bs_context_enable_timing", fp.ctx, 0)
    fp.close()
