"""Selector evidence (SURVEY S-1, src/adaptive.cpp:16-32): search for a regime
where the pixel-wise SharedMemOpt baseline beats FineGrainedCombined on B200,
and record what the per-frame predictor (bs_select_variant) and the
reference's checkpoint rule (switch when t_balanced > t_baseline) choose.

Grid: resolution x Gaussian count x opacity scale x patch size x clustering.
Per point: render times of FineGrainedCombined, SharedMemOpt and Naive on the
point's TileBinning, each launch from a flushed L2 (256 MiB write, outside the
timed interval), median of 5; the selector's pick; regret.

  python tools/selector_sweep.py --out profiles/r2_selector_sweep.jsonl
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

RES = [(256, 256, 256.0), (1920, 1080, 1000.0), (3840, 2160, 2000.0)]
COUNTS = [1_000, 10_000, 100_000, 1_000_000]
OPACITY = [1.0, 0.1]
PATCH = [(16, 16), (8, 8)]
GEOM = [(1.0, 0.035), (0.12, 0.035)]  # uniform, clustered


def timed(fn, flush, reps=5):
    fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    res = RES[:2] if a.quick else RES
    with open(a.out, "w") as fo:
        for W, H, f in res:
            for n in COUNTS:
                if n * 56 > 8 << 30:
                    continue
                for bgf, sig in GEOM:
                    cam = api.camera(None, (f, f), W, H)
                    g3d0 = api.gen_clustered_scene(n, cam, cluster_sigma=sig, background_fraction=bgf)
                    for osc in OPACITY:
                        g3d = g3d0.copy()
                        g3d["opacity"] *= np.float32(osc)
                        d = api.g3d_to_device(g3d)
                        for pw, ph in PATCH:
                            pipe = api.Pipeline(W, H, pw, ph, "cuda", N.ALPHA_EXACT)
                            frame, v_auto = pipe.forward(d, n, cam, variant="auto")
                            s, b, st = pipe.splats, pipe.last_binning, pipe.last_stats
                            ms = {}
                            for v in (3, 4, 0):
                                ms[api.variant_name(v)] = round(timed(
                                    lambda v=v: api.render_forward(v, s, b, W, H, pw, ph, (0, 0, 0), N.ALPHA_EXACT,
                                                                   st.task_order, frame, pipe.render_ws), flush), 5)
                            summ = st.summary()
                            best = min(ms.values())
                            pick = api.variant_name(v_auto)
                            rec = {"W": W, "H": H, "n": n, "background_fraction": bgf, "cluster_sigma": sig,
                                   "opacity_scale": osc, "patch": [pw, ph], "K": b.k, "tile_max": summ["max"],
                                   "tile_mean": round(summ["mean"], 2), "render_ms_l2_flushed": ms,
                                   "selector": pick, "selector_regret": round(ms[pick] / best - 1.0, 4)
                                   if pick in ms else None,
                                   "checkpoint_switches": ms["FineGrainedCombined"] > ms["SharedMemOpt"],
                                   "smo_over_fg": round(ms["FineGrainedCombined"] / ms["SharedMemOpt"], 3)}
                            fo.write(json.dumps(rec) + "\n")
                            fo.flush()
                            print(json.dumps(rec), flush=True)
                            del pipe, frame, s, b, st
                        del d
                    torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
