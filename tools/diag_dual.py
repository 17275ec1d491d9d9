"""Two frame contexts on two streams, views alternating (diagnostic): does
view i+1's preprocess/binning overlap view i's render?"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2412_17378_b200 import api  # noqa: E402

W, H, f, n = 1920, 1080, 1000.0, 1_000_000
cams = [api.camera(bench.orbit_view(k), (f, f), W, H) for k in range(64)]
g3d = api.gen_clustered_scene(n, cams[0])
d = api.g3d_to_device(g3d, "cuda")
for nctx in (1, 2, 3):
    streams = [torch.cuda.Stream() for _ in range(nctx)]
    flush = [torch.empty(256 << 20, dtype=torch.uint8, device="cuda") for _ in range(nctx)]
    fps = []
    for s in streams:
        with torch.cuda.stream(s):
            fps.append(api.FramePipeline(W, H, 16, 16, "cuda", 0, async_mode=True, graphs=True))
    for i in range(12):
        with torch.cuda.stream(streams[i % nctx]):
            fps[i % nctx].forward(d, n, cams[i % 64])
    for fp in fps:
        fp.sync()
    torch.cuda.synchronize()
    steps = 192
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record()
    for s in streams:
        s.wait_stream(torch.cuda.current_stream())
    for i in range(steps):
        with torch.cuda.stream(streams[i % nctx]):
            if os.environ.get("FLUSH") == "1":
                flush[i % nctx].zero_()
            fps[i % nctx].forward(d, n, cams[(12 + i) % 64])
    for fp in fps:
        fp.sync()
    for s in streams:
        torch.cuda.current_stream().wait_stream(s)
    end.record()
    torch.cuda.synchronize()
    ms = start.elapsed_time(end) / steps
    print(f"contexts {nctx}: {ms:.3f} ms/view, {1000 / ms:.1f} views/s", flush=True)
    for fp in fps:
        fp.close()
