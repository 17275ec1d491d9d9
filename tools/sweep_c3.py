"""C3: imbalance sweep on the C2 geometry (1080p, 1M Gaussians) — render time
of every variant in both alpha modes, tile-work statistics, the per-frame
selector's choice and its regret  t(chosen) / min_v t(v) - 1.

Axis 1 (geometric): background_fraction 1.0 -> 0.05 with
cluster_sigma 0.035 -> 0.02 (uniform -> clustered).
Axis 2 (training stage): opacity scaled by s in {1, 0.5, 0.25, 0.1, 0.05} on
the most clustered geometry — early 3DGS training (low opacities, long
per-pixel consumption) is where the paper's imbalance lives.

  python tools/sweep_c3.py [--out profiles/r1_c3_sweep.jsonl] [--quick]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2412_17378_b200 import _native as N  # noqa: E402
from paper_2412_17378_b200 import api  # noqa: E402

GEOM = [(1.0, 0.035), (0.8, 0.032), (0.6, 0.03), (0.4, 0.027), (0.25, 0.025), (0.12, 0.022), (0.05, 0.02)]
OPACITY = [1.0, 0.5, 0.25, 0.1, 0.05]


def time_render(v, m, s, b, st, frame, W, H, reps=5):
    api.render_forward(v, s, b, W, H, 16, 16, (0, 0, 0), m, st.task_order, frame)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, e in ev:
        a.record()
        api.render_forward(v, s, b, W, H, 16, 16, (0, 0, 0), m, st.task_order, frame)
        e.record()
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(e) for a, e in ev]))


def point(bgf, sigma, oscale, n=1_000_000, W=1920, H=1080, f=1000.0, n_clusters=4):
    cam = api.camera(None, (f, f), W, H)
    g3d = api.gen_clustered_scene(n, cam, n_clusters=n_clusters, cluster_sigma=sigma, background_fraction=bgf)
    g3d["opacity"] *= oscale
    pipe = api.Pipeline(W, H, 16, 16, "cuda", N.ALPHA_EXACT)
    frame, _ = pipe.forward(api.g3d_to_device(g3d), n, cam, variant=0)
    s, b, st = pipe.splats, pipe.last_binning, pipe.last_stats
    E, C = api.frame_work(frame, b, 16, 16)
    term = frame.term.cpu().numpy().reshape(H, W)
    rg = b.tile_ranges.cpu().numpy().view(np.uint32)
    rows, cols = (H + 15) // 16, (W + 15) // 16
    lens = (rg[1::2] - rg[0::2]).astype(np.int64).reshape(rows, cols)
    full = np.repeat(np.repeat(lens, 16, 0), 16, 1)[:H, :W]
    cons = np.where(term > 0, term, full)
    pad = np.zeros((rows * 16, cols * 16), np.int64)
    pad[:H, :W] = cons
    tile_work = pad.reshape(rows, 16, cols, 16).sum(axis=(1, 3))
    out = {"n": n, "W": W, "H": H, "n_clusters": n_clusters, "bgf": bgf, "sigma": sigma, "opacity_scale": oscale, "K": b.k, "E": E, "C": C,
           "list_max": int(lens.max()), "list_mean": float(lens.mean()),
           "tile_work_max": int(tile_work.max()), "tile_work_mean": float(tile_work.mean()),
           "work_imbalance": float(tile_work.max() / max(1.0, tile_work.mean())),
           "selector": api.variant_name(api.select_variant(st, W, H, 16, 16))}
    for m, mn in ((N.ALPHA_EXACT, "exact"), (N.ALPHA_FAST, "fast")):
        t = {api.variant_name(v): round(time_render(v, m, s, b, st, frame, W, H), 4) for v in range(5)}
        out[f"ms_{mn}"] = t
        best = min(t.values())
        out[f"regret_{mn}"] = round(t[out["selector"]] / best - 1.0, 4)
        out[f"fg_vs_naive_{mn}"] = round(t["Naive"] / t["FineGrainedCombined"], 3)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "c3_sweep.jsonl"))
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--extreme", action="store_true", help="single-cluster extremes + C1")
    a = ap.parse_args()
    pts = [(g, s, 1.0) for g, s in GEOM] + [(GEOM[-1][0], GEOM[-1][1], o) for o in OPACITY[1:]]
    if a.quick:
        pts = pts[:2] + pts[-2:]
    extra = []
    if a.extreme:
        pts = []
        extra = [dict(bgf=0.05, sigma=0.01, oscale=o, n_clusters=1) for o in (1.0, 0.25, 0.05, 0.02)]
        extra += [dict(bgf=1.0, sigma=0.035, oscale=1.0, n=10_000, W=256, H=256, f=256.0)]
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as fh:
        for kw in [dict(bgf=g, sigma=s_, oscale=o) for g, s_, o in pts] + extra:
            r = point(**kw)
            fh.write(json.dumps(r) + "\n")
            fh.flush()
            print(json.dumps({k: r[k] for k in ("n", "n_clusters", "bgf", "sigma", "opacity_scale", "work_imbalance",
                                                 "selector", "regret_exact", "fg_vs_naive_exact", "fg_vs_naive_fast",
                                                 "ms_exact")}), flush=True)


if __name__ == "__main__":
    main()
