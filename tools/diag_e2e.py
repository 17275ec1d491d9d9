"""e2e pipeline timing: with / without downloads (diagnostic)."""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2412_17378_b200 import _native as N  # noqa: E402
from paper_2412_17378_b200 import api  # noqa: E402

W, H, f, n = 1920, 1080, 1000.0, int(os.environ.get("NG", "1000000"))
cams = [api.camera(bench.orbit_view(k), (f, f), W, H) for k in range(64)]
g3d = api.gen_clustered_scene(n, cams[0])
host = torch.from_numpy(np.ascontiguousarray(g3d).view(np.uint8).reshape(-1).copy()).pin_memory()
P = W * H
rings = [[torch.empty(3 * P, dtype=torch.float32).pin_memory()] +
         [torch.empty(P, dtype=torch.float32).pin_memory() for _ in range(3)] +
         [torch.empty(P, dtype=torch.int32).pin_memory() for _ in range(2)] for _ in range(3)]
bg = (C.c_float * 3)(0, 0, 0)
ctx = C.c_void_p()
N.call("bs_context_create", C.byref(ctx), 0)
N.call("bs_context_set_async", ctx, 1)
for mode in ("full", "no_d2h", "color_only", "full"):
    def step(k):
        outs = rings[k % 3]
        ptrs = [o.data_ptr() for o in outs]
        if mode == "no_d2h":
            ptrs = [None] * 6
        elif mode == "color_only":
            ptrs = [ptrs[0]] + [None] * 5
        N.call("bs_render_frame_host_async", ctx, host.data_ptr(), n, C.byref(cams[k % 64]), 16, 16, -1, bg, *ptrs)
    for k in range(4):
        step(k)
    N.call("bs_context_sync", ctx, None)
    host_t = []
    t0 = time.perf_counter()
    for k in range(30):
        a = time.perf_counter()
        step(k)
        host_t.append(time.perf_counter() - a)
    N.call("bs_context_sync", ctx, None)
    dt = (time.perf_counter() - t0) / 30
    print(f"{mode}: {dt * 1e3:.3f} ms/frame; host call p50 {np.median(host_t) * 1e3:.3f} ms")
