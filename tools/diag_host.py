"""Host (CPU) cost of each C-ABI stage call, GPU left running (diagnostic)."""
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

W, H, f, n = 1920, 1080, 1000.0, 1_000_000
cam = api.camera(bench.orbit_view(0), (f, f), W, H)
g3d = api.gen_clustered_scene(n, cam)
d = api.g3d_to_device(g3d, "cuda")
pipe = api.Pipeline(W, H, 16, 16, "cuda", 0)
frame, v = pipe.forward(d, n, cam)
torch.cuda.synchronize()
s, b = pipe.splats, pipe.last_binning
st = pipe.last_stats
L = N.lib()
T = b.tile_count
rg = b.tile_ranges
hist = torch.zeros(64, dtype=torch.uint8, device="cuda")
order = torch.empty(T, dtype=torch.int32, device="cuda")
sm = api._stream("cuda")
res = {}


def tm(name, fn, reps=50):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
        torch.cuda.synchronize()
    res[name] = np.median(ts) * 1e6


tm("preprocess", lambda: api.project_all(d, n, cam, pipe.splats, pipe.pre_ws))
tm("bin_count", lambda: pipe.binner.count(s))
tm("bin_sort", lambda: pipe.binner.sort(s, b.k))
tm("tile_order", lambda: L.bs_tile_order(rg.data_ptr(), T, hist.data_ptr(), order.data_ptr(), sm))
tm("render_fg", lambda: api.render_forward(3, s, b, W, H, 16, 16, (0, 0, 0), 0, st.task_order, frame))
tm("render_smo", lambda: api.render_forward(4, s, b, W, H, 16, 16, (0, 0, 0), 0, st.task_order, frame))
tm("occupancy_only", lambda: L.bs_device_sm_count(C.byref(C.c_int32())))
tm("null_ctypes", lambda: L.bs_abi_version())
for k, v in res.items():
    print(f"{k:16s} host {v:9.1f} us")
