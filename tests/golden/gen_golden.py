"""Freeze FNV-1a digests (include/splatsim/rng.hpp:60-69) of the oracle's
outputs on fixed fixtures -> tests/golden/digests.json.

The reference's own frozen fixture digest (include/splatsim/experiment.hpp:13-15)
is not in the mount, so these are regenerated from the restated oracle and
then frozen: any later change to the oracle (or to its inputs) that alters a
single bit of these fixtures fails tests/test_golden.py.

  python tests/golden/gen_golden.py      # rewrite digests.json
"""
from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

import oracle_lib as O  # noqa: E402

FIXTURES = {
    # name: (n, W, H, f, bgfrac, pw, ph, bg)
    "c1_uniform_256": (10000, 256, 256, 256.0, 1.0, 16, 16, (0.0, 0.0, 0.0)),
    "clustered_192x128_16x8": (6000, 192, 128, 192.0, 0.12, 16, 8, (0.1, 0.2, 0.3)),
    "clustered_64x64": (200, 64, 64, 64.0, 0.5, 16, 16, (0.1, 0.2, 0.3)),
}


def compute() -> dict:
    out = {}
    for name, (n, W, H, f, bgf, pw, ph, bg) in FIXTURES.items():
        cam = O.make_camera(focal=(f, f), width=W, height=H)
        g3d = O.gen_clustered_scene(n, cam, bgfrac=bgf)
        g2d = O.project_all(g3d, cam)
        pl, rg = O.bin_tiles(g2d, W, H, pw, ph)
        d = {"n_visible": int(len(g2d)), "K": int(len(pl)), "g3d": O.fnv1a64(g3d), "g2d": O.fnv1a64(g2d),
             "point_list": O.fnv1a64(pl), "tile_ranges": O.fnv1a64(rg)}
        for v, tag in ((0, "render_reference"), (2, "render_gaussianwise")):
            r = O.render(v, pl, rg, g2d, W, H, pw, ph, bg, lazy=True, threads=0)
            d[tag] = {k: O.fnv1a64(r[k]) for k in ("color", "alpha", "depth", "final_t", "contrib", "term")}
        out[name] = d
    return out


if __name__ == "__main__":
    with open(os.path.join(HERE, "digests.json"), "w") as f:
        json.dump(compute(), f, indent=1, sort_keys=True)
    print("wrote", os.path.join(HERE, "digests.json"))
