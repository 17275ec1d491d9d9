"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
C1 (256x256, 10k Gaussians) through every variant on the API path (exact and
fast), a 1 Mpixel frame through the frame pipeline (fused projection,
super-tile lists, device-selected variant, async K checks, CUDA-graph
replays), the FineGrainedCombined tail hand-off forced on, and the host-buffer
pipeline — each output checked against the oracle, so a sanitizer-clean run
is also a correct one.

  compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
os.environ.setdefault("BS_FINE_DONATE_AFTER", "32")  # exercise the tail hand-off (k_render_donated)
os.environ.setdefault("BS_FINE_DONATE_MIN", "64")
import oracle_lib as O  # noqa: E402
from paper_2412_17378_b200 import _native as N  # noqa: E402
from paper_2412_17378_b200 import api  # noqa: E402


def check(got, ref, exact_colour):
    assert np.array_equal(got["contrib"], ref["contrib"]) and np.array_equal(got["term"], ref["term"])
    assert np.array_equal(got["final_t"], ref["final_t"])
    err = float(np.abs(got["color"] - ref["color"]).max())
    assert err == 0.0 if exact_colour else err <= 1e-6, err


def main():
    W = H = 256
    cam = O.make_camera(focal=(256.0, 256.0), width=W, height=H)
    g3d = O.gen_clustered_scene(10000, cam, bgfrac=1.0)
    g2d = O.project_all(g3d, cam)
    pl, rg = O.bin_tiles(g2d, W, H, 16, 16)
    bg = (0.1, 0.2, 0.3)
    refs = {v: O.render(v, pl, rg, g2d, W, H, 16, 16, bg, lazy=True, threads=0) for v in (0, 2)}
    pipe = api.Pipeline(W, H, 16, 16, "cuda", N.ALPHA_EXACT)
    d = api.g3d_to_device(g3d)
    for mode in (N.ALPHA_EXACT, N.ALPHA_FAST):
        pipe.alpha_mode = mode
        for v in range(5):
            f, _ = pipe.forward(d, len(g3d), N.Camera.from_buffer_copy(bytes(cam)), variant=v, bg=bg)
            torch.cuda.synchronize()
            if mode == N.ALPHA_EXACT:
                check(f.to_numpy(), refs[2 if v == 2 else 0], v in (0, 1, 4))
    print("C1 API path: 5 variants x 2 modes ok", flush=True)
    # backward render on C1, both alpha modes; exact vs the oracle
    rng = np.random.default_rng(0)
    P = W * H
    dl = [rng.normal(size=k * P).astype(np.float32) for k in (3, 1, 1)]
    gref = O.render_backward(pl, rg, g2d, W, H, 16, 16, bg, *dl)
    s = api.splats_from_g2d(g2d, "cuda")
    b = api.bin_tiles(s, W, H, 16, 16)
    for mode in (N.ALPHA_EXACT, N.ALPHA_FAST):
        f = api.render_forward(3, s, b, W, H, 16, 16, bg, mode)
        g = api.render_backward(s, b, f, W, H, 16, 16, *[torch.from_numpy(x).cuda() for x in dl], bg=bg,
                                alpha_mode=mode)
        torch.cuda.synchronize()
        if mode == N.ALPHA_EXACT:
            got = g.as_fields()[: len(g2d)].double().cpu().numpy()
            scale = np.maximum(1.0, np.abs(gref).max(axis=0))
            assert (np.abs(got - gref).max(axis=0) <= 2e-4 * scale).all()
    print("C1 backward render: 2 modes ok", flush=True)
    # frame pipeline at 1 Mpixel (super-tile lists), async + graphs
    W = H = 1024
    cam = O.make_camera(focal=(1024.0, 1024.0), width=W, height=H)
    g3d = O.gen_clustered_scene(20000, cam)
    g2d = O.project_all(g3d, cam)
    pl, rg = O.bin_tiles(g2d, W, H, 16, 16)
    ref = O.render(0, pl, rg, g2d, W, H, 16, 16, bg, lazy=True, threads=0)
    fp = api.FramePipeline(W, H, 16, 16, "cuda", N.ALPHA_EXACT, async_mode=True, graphs=True, fine_ctas=3)
    d = api.g3d_to_device(g3d)
    ncam = N.Camera.from_buffer_copy(bytes(cam))
    for _ in range(4):
        fp.forward(d, len(g3d), ncam, variant="auto", bg=bg)
    fp.sync()
    check(fp.frame.to_numpy(), ref, False)
    fp.close()
    print("frame pipeline 1024x1024 (super-tile lists, async, graphs): ok", flush=True)
    # host-buffer pipeline
    ctx = N.C.c_void_p()
    N.call("bs_context_create", N.C.byref(ctx), N.ALPHA_EXACT)
    N.call("bs_context_set_async", ctx, 1)
    P = W * H
    outs = [np.zeros(3 * P, np.float32)] + [np.zeros(P, np.float32) for _ in range(3)] + \
           [np.zeros(P, np.int32) for _ in range(2)]
    bgc = (N.C.c_float * 3)(*bg)
    for _ in range(3):
        N.call("bs_render_frame_host_async", ctx, g3d.ctypes.data, len(g3d), N.C.byref(ncam), 16, 16, -1, bgc,
               *[o.ctypes.data for o in outs])
    N.call("bs_context_sync", ctx, None)
    N.call("bs_context_destroy", ctx)
    got = dict(zip(("color", "alpha", "depth", "final_t", "contrib", "term"), outs))
    check(got, ref, False)
    print("host-buffer pipeline: ok", flush=True)


if __name__ == "__main__":
    main()
