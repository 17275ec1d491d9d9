"""Exploration: per-variant render time vs scene regime (opacity scale,
cluster sigma) on the C2 geometry.  Prints one JSON line per scene."""
from __future__ import annotations

import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2412_17378_b200 import _native as N  # noqa: E402
from paper_2412_17378_b200 import api  # noqa: E402


def run(opacity_scale=1.0, sigma=0.035, bgf=0.12, n=1_000_000, W=1920, H=1080, f=1000.0, modes=(0, 1), reps=3):
    cam = api.camera(None, (f, f), W, H)
    g3d = api.gen_clustered_scene(n, cam, cluster_sigma=sigma, background_fraction=bgf)
    g3d["opacity"] *= opacity_scale
    d = api.g3d_to_device(g3d)
    pipe = api.Pipeline(W, H, 16, 16, "cuda", 0)
    frame, _ = pipe.forward(d, n, cam, variant=0)
    s, b, st = pipe.splats, pipe.last_binning, pipe.last_stats
    res = {"opacity_scale": opacity_scale, "sigma": sigma, "bgf": bgf, "K": b.k, "stats": st.summary()}
    for m in modes:
        times = {}
        for v in range(5):
            api.render_forward(v, s, b, W, H, 16, 16, (0, 0, 0), m, st.task_order, frame)
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
            for a, e in ev:
                a.record()
                api.render_forward(v, s, b, W, H, 16, 16, (0, 0, 0), m, st.task_order, frame)
                e.record()
            torch.cuda.synchronize()
            times[N.VARIANTS[v]] = round(float(np.mean([a.elapsed_time(e) for a, e in ev])), 3)
        res[f"ms_mode{m}"] = times
    api.render_forward(0, s, b, W, H, 16, 16, (0, 0, 0), 0, st.task_order, frame)
    E, Cc = api.frame_work(frame, b, 16, 16)
    term = frame.term.cpu().numpy().reshape(H, W)
    rg = b.tile_ranges.cpu().numpy().view(np.uint32)
    lens = (rg[1::2] - rg[0::2]).astype(np.int64).reshape(68, 120)
    cons = np.where(term > 0, term, np.repeat(np.repeat(lens, 16, 0), 16, 1)[:H, :W])
    tw = cons[: 68 * 16 - 8].reshape(-1)  # not exact per tile; report pixel stats
    tile_work = np.zeros((68, 120))
    for ty in range(68):
        for tx in range(120):
            tile_work[ty, tx] = cons[ty * 16:(ty + 1) * 16, tx * 16:(tx + 1) * 16].sum()
    res.update({"E": E, "C": Cc, "E_per_px": E / (W * H), "max_px_consumed": int(cons.max()),
                "p99_px_consumed": float(np.percentile(cons, 99)), "max_tile_work": float(tile_work.max()),
                "mean_tile_work": float(tile_work.mean()), "frac_px_unterminated": float((term == 0).mean())})
    del tw
    return res


if __name__ == "__main__":
    for osc, sig in [(1.0, 0.035), (0.5, 0.035), (0.25, 0.035), (0.1, 0.035), (0.1, 0.015), (0.25, 0.015),
                     (1.0, 0.015)]:
        print(json.dumps(run(osc, sig)), flush=True)
