"""Does a concurrent PCIe copy slow the frame's kernels? (diagnostic)
Frames on one context (device input), with a side stream copying in a loop:
none / D2H 66 MB / D2H 8 MB (L2-resident source) / H2D 56 MB."""
import os
import sys
import threading

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
fp = api.FramePipeline(W, H, 16, 16, "cuda", 0, async_mode=True)
for i in range(8):
    fp.forward(d, n, cams[i % 64])
fp.sync()
side = torch.cuda.Stream()
big_d, big_h = torch.empty(66 << 20, dtype=torch.uint8, device="cuda"), torch.empty(66 << 20, dtype=torch.uint8).pin_memory()
sm_d, sm_h = torch.empty(8 << 20, dtype=torch.uint8, device="cuda"), torch.empty(8 << 20, dtype=torch.uint8).pin_memory()
up_h, up_d = torch.empty(56 << 20, dtype=torch.uint8).pin_memory(), torch.empty(56 << 20, dtype=torch.uint8, device="cuda")
modes = {"none": None, "d2h66": lambda: big_h.copy_(big_d, non_blocking=True),
         "d2h8x8": lambda: [sm_h.copy_(sm_d, non_blocking=True) for _ in range(8)],
         "h2d56": lambda: up_d.copy_(up_h, non_blocking=True)}
for name, fn in list(modes.items()) * 2:
    N.call("bs_context_enable_timing", fp.ctx, 1)
    if fn:
        with torch.cuda.stream(side):
            for _ in range(60):
                fn()
    st = []
    for i in range(20):
        fp.forward(d, n, cams[(8 + i) % 64])
        fp.sync()
        st.append(list(fp.stage_ms().values()))
    torch.cuda.synchronize()
    N.call("bs_context_enable_timing", fp.ctx, 0)
    m = np.mean(st, axis=0)
    print(f"{name:8s} stages {np.round(m, 3).tolist()} sum {m.sum():.3f}")
