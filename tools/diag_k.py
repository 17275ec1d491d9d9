import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2412_17378_b200 import api
W, H, f, n = 1920, 1080, 1000.0, 1_000_000
cams = [api.camera(bench.orbit_view(k), (f, f), W, H) for k in range(64)]
g3d = api.gen_clustered_scene(n, cams[0])
d = api.g3d_to_device(g3d, "cuda")
fp = api.FramePipeline(W, H, 16, 16, "cuda", 0, async_mode=True)
ks = []
for i in range(64):
    _, fi = fp.forward(d, n, cams[i], info=True)
    ks.append(fi.k)
    print(i, fi.k, fp.capacity(), flush=True)
