"""FG render timing on the C2 identity view three ways (diagnostic): events
around each call, events around 20 back-to-back calls, and the kernels only
(ncu gives the per-kernel durations of the same calls)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2412_17378_b200 import _native as N  # noqa: E402
from paper_2412_17378_b200 import api  # noqa: E402

W, H, f, n, bgf, sig = bench.CONFIGS["c2"]
cam = api.camera(np.eye(4, dtype=np.float32), (f, f), W, H)
g3d = api.gen_clustered_scene(n, cam, cluster_sigma=sig, background_fraction=bgf)
d = api.g3d_to_device(g3d)
pipe = api.Pipeline(W, H, 16, 16, "cuda", N.ALPHA_EXACT)
frame, v = pipe.forward(d, n, cam, variant="FineGrainedCombined")
s, b, st = pipe.splats, pipe.last_binning, pipe.last_stats
stream = torch.cuda.current_stream()


VARIANT = api.variant_from_name(os.environ.get("DIAG_VARIANT", "FineGrainedCombined"))


def call():
    api.render_forward(VARIANT, s, b, W, H, 16, 16, (0, 0, 0), N.ALPHA_EXACT, st.task_order, frame, pipe.render_ws)


for _ in range(3):
    call()
torch.cuda.synchronize()
per = []
for _ in range(10):
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    call()
    e.record(stream)
    torch.cuda.synchronize()
    per.append(a.elapsed_time(e))
a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(stream)
for _ in range(20):
    call()
e.record(stream)
torch.cuda.synchronize()
print(f"per-call events (synced): median {np.median(per):.4f} ms; 20 back-to-back: {a.elapsed_time(e) / 20:.4f} ms/call")

# backward render on the same frame (random dL; grads accumulate, zeroed once)
if os.environ.get("DIAG_BWD", "1") == "1":
    g = torch.Generator(device="cuda").manual_seed(3)
    P = W * H
    dl = (torch.rand(3 * P, device="cuda", generator=g) - 0.5, torch.rand(P, device="cuda", generator=g) - 0.5,
          torch.rand(P, device="cuda", generator=g) - 0.5)
    grads = api.SplatGrads.zeros(s.n_cap, "cuda")

    def bcall():
        api.render_backward(s, b, frame, W, H, 16, 16, dl[0], dl[1], dl[2], (0, 0, 0), N.ALPHA_EXACT, st.task_order,
                            grads, pipe.render_ws)

    for _ in range(3):
        bcall()
    torch.cuda.synchronize()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(10):
        bcall()
    e.record(stream)
    torch.cuda.synchronize()
    print(f"backward: {a.elapsed_time(e) / 10:.4f} ms/call")
