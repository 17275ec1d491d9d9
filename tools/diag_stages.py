"""Per-stage device times of the frame pipeline (one context, L2 flushed
between frames), mean over 60 frames of the C2 orbit (diagnostic)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2412_17378_b200 import _native as N  # noqa: E402
from paper_2412_17378_b200 import api  # noqa: E402
from paper_2412_17378_b200 import sharding  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
W, H, f, n, bgf, sig = bench.CONFIGS[cfg]
cams = [api.camera(sharding.orbit_view(k), (f, f), W, H) for k in range(64)]
g3d = api.gen_clustered_scene(n, cams[0], cluster_sigma=sig, background_fraction=bgf)
d = api.g3d_to_device(g3d, "cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
fp = api.FramePipeline(W, H, 16, 16, "cuda", 0, async_mode=True)
for i in range(10):
    fp.forward(d, n, cams[i % 64])
fp.sync()
N.call("bs_context_enable_timing", fp.ctx, 1)
stages = []
for i in range(60):
    flush.zero_()
    fp.forward(d, n, cams[(10 + i) % 64])
    fp.sync()
    torch.cuda.synchronize()
    stages.append(list(fp.stage_ms().values()))
st = np.mean(stages, axis=0)
print(f"{os.environ.get('TAG', '')} {cfg}: stages {dict(zip(fp.stage_ms().keys(), np.round(st, 4).tolist()))} sum {st.sum():.4f}")
