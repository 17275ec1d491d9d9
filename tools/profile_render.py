"""Render one C2 frame with a chosen variant/mode (for ncu captures).

  python tools/profile_render.py --variant Naive --alpha exact [--opacity-scale 0.1 --sigma 0.015] [--reps 2]
"""
from __future__ import annotations

import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2412_17378_b200 import api  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variant", default="Naive")
    ap.add_argument("--alpha", default="exact")
    ap.add_argument("--opacity-scale", type=float, default=1.0)
    ap.add_argument("--sigma", type=float, default=0.035)
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--W", type=int, default=1920)
    ap.add_argument("--H", type=int, default=1080)
    ap.add_argument("--f", type=float, default=1000.0)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--config", default=None, help="c1/c2/c4: bench.py's scene and first view (overrides n/W/H/f/sigma)")
    ap.add_argument("--frame-pipeline", action="store_true",
                    help="render through the frame pipeline (super-tile lists on >= 1 Mpixel frames)")
    ap.add_argument("--backward", action="store_true",
                    help="after the forward, run bs_render_backward (random dL) --reps times")
    ap.add_argument("--fine-ctas", type=int, default=0,
                    help="FineGrainedCombined CTAs per SM (bs_render_set_fine_occupancy; the bench's timed frames use 3)")
    a = ap.parse_args()
    if a.fine_ctas:
        from paper_2412_17378_b200 import _native as N
        N.call("bs_render_set_fine_occupancy", a.fine_ctas)
    if a.config:
        import bench
        a.W, a.H, a.f, a.n, bgf, a.sigma = bench.CONFIGS[a.config]
        cam = api.camera(bench.orbit_view(0), (a.f, a.f), a.W, a.H)
        g3d = api.gen_clustered_scene(a.n, cam, cluster_sigma=a.sigma, background_fraction=bgf)
    else:
        cam = api.camera(None, (a.f, a.f), a.W, a.H)
        g3d = api.gen_clustered_scene(a.n, cam, cluster_sigma=a.sigma)
    g3d["opacity"] *= a.opacity_scale
    mode = 0 if a.alpha == "exact" else 1
    d = api.g3d_to_device(g3d)
    v = api.variant_from_name(a.variant)
    if a.frame_pipeline:
        fp = api.FramePipeline(a.W, a.H, 16, 16, "cuda", mode)
        for _ in range(a.reps):
            fp.forward(d, a.n, cam, variant=v)
        fp.sync()
    else:
        pipe = api.Pipeline(a.W, a.H, 16, 16, "cuda", mode)
        for _ in range(1 if a.backward else a.reps):
            frame, _ = pipe.forward(d, a.n, cam, variant=v)
        if a.backward:
            P = a.W * a.H
            dl = [torch.randn(k * P, device="cuda") for k in (3, 1, 1)]
            for _ in range(a.reps):
                api.render_backward(pipe.splats, pipe.last_binning, frame, a.W, a.H, 16, 16, dl[0], dl[1], dl[2],
                                    alpha_mode=mode, task_order=pipe.last_stats.task_order, ws=pipe.render_ws)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
