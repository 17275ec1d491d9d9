"""Potential of CUDA-graph replay for the frame (diagnostic): the same view
rendered N times (a) through bs_render_frame_device, (b) as a captured graph."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2412_17378_b200 import _native as N  # noqa: E402
from paper_2412_17378_b200 import api  # noqa: E402

W, H, f, n = 1920, 1080, 1000.0, 1_000_000
cam = api.camera(bench.orbit_view(20), (f, f), W, H)
g3d = api.gen_clustered_scene(n, cam)
d = api.g3d_to_device(g3d, "cuda")
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    fp = api.FramePipeline(W, H, 16, 16, "cuda", 0, async_mode=True)
    for _ in range(6):
        fp.forward(d, n, cam)
    fp.sync()
    s.synchronize()
    reps = 50
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fp.forward(d, n, cam)
    b.record()
    fp.sync()
    s.synchronize()
    t_plain = a.elapsed_time(b) / reps
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        N.call("bs_context_set_stream", fp.ctx, s.cuda_stream)
        fp.forward(d, n, cam)
    N.call("bs_context_drop_pending", fp.ctx)  # the captured frame's K check never ran
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(reps):
    g.replay()
b.record()
torch.cuda.synchronize()
t_graph = a.elapsed_time(b) / reps
print(f"plain {t_plain:.3f} ms/frame, graph {t_graph:.3f} ms/frame")
