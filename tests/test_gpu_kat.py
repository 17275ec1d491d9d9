"""SPEC known-answer tests of the blending rows (eval_alpha,
blend_pixel, termination_index, the Gaussian-wise blend), run on the device
through every render variant: splats are placed so one pixel sees exactly
the KAT's step list, and the pixel's outputs are checked against the KAT
value AND bit-exactly against the oracle's render of the same splats.

  R1 eval_alpha       src/blend.cpp:8-14
  R2 blend_pixel      src/blend.cpp:16-42
  R3 termination_index src/blend.cpp:44-53
  R5/R6 Gaussian-wise src/kernels.cpp:57-107, inc/blend.hpp:69-83
"""
from __future__ import annotations

import math

import numpy as np
import pytest

import oracle_lib as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from paper_2412_17378_b200 import _native as N  # noqa: E402
from paper_2412_17378_b200 import api  # noqa: E402

W, H, PW, PH = 32, 16, 16, 16
PX, PY = 5, 7  # the probed pixel: sample point (5.5, 7.5)


def splat(x, y, opacity, color, depth, conic=(1e-6, 0.0, 1e-6), radius=2.0):
    g = np.zeros(1, dtype=O.G2D_DTYPE)
    g["x"], g["y"] = x, y
    g["conic_a"], g["conic_b"], g["conic_c"] = conic
    g["opacity"], g["color"], g["depth"], g["radius"] = opacity, color, depth, radius
    return g


def render_all(g2d, bg):
    """Every variant's frame on the device + the oracle's, bit-compared."""
    pl, rg = O.bin_tiles(g2d, W, H, PW, PH)
    out = {}
    for v in range(5):
        s = api.splats_from_g2d(g2d, "cuda")
        b = api.bin_tiles(s, W, H, PW, PH)
        st = api.tile_load_histogram(b)
        got = api.render_forward(v, s, b, W, H, PW, PH, bg, N.ALPHA_EXACT, st.task_order).to_numpy()
        ref = O.render(v, pl, rg, g2d, W, H, PW, PH, bg, lazy=True, threads=0)
        for k in ("contrib", "term"):
            assert np.array_equal(got[k], ref[k]), (v, k)
        for k in ("final_t", "alpha"):
            assert np.array_equal(got[k].view(np.uint32), ref[k].view(np.uint32)), (v, k)
        for k in ("color", "depth"):
            if v in (0, 1, 4):  # pixel-wise: serial double sums, bit-exact
                assert np.array_equal(got[k].view(np.uint32), ref[k].view(np.uint32)), (v, k)
            else:  # Gaussian-wise: the same terms summed in a different order (S17 max_rel)
                assert np.max(np.abs(got[k] - ref[k]) / np.maximum(1, np.abs(ref[k]))) <= 1e-6, (v, k)
        out[v] = got
    return out


def pix(f, k):
    i = PY * W + PX
    return f[k].reshape(H * W, -1)[i] if k == "color" else f[k].reshape(-1)[i]


def test_eval_alpha_center_is_clamped_opacity():
    # d = 0 -> alpha = min(0.99, opacity)
    for op, want in ((0.7, np.float32(0.7)), (1.0, np.float32(0.99))):
        g = splat(PX + 0.5, PY + 0.5, op, (1, 1, 1), 1.0)
        for f in render_all(g, (0, 0, 0)).values():
            assert pix(f, "contrib") == 1
            assert pix(f, "final_t") == np.float32(1) * (np.float32(1) - want)


def test_eval_alpha_conic_exp_minus_two():
    # conic (1, 0, 1), opacity 1, d = (2, 0) -> power -2, alpha = e^-2
    g = splat(PX + 0.5 + 2.0, PY + 0.5, 1.0, (1, 0, 0), 1.0, conic=(1.0, 0.0, 1.0), radius=3.0)
    for f in render_all(g, (0, 0, 0)).values():
        a = 1.0 - float(pix(f, "final_t"))
        assert abs(a - math.exp(-2.0)) < 1e-6
        assert pix(f, "contrib") == 1


def test_blend_pixel_three_half_steps():
    # three alpha = 0.5 steps R, G, B, bg 0 -> (0.5, 0.25, 0.125), T 0.125, contrib 3
    g = np.concatenate([splat(PX + 0.5, PY + 0.5, 0.5, c, d) for c, d in
                        (((1, 0, 0), 1.0), ((0, 1, 0), 2.0), ((0, 0, 1), 3.0))])
    for f in render_all(g, (0, 0, 0)).values():
        assert np.allclose(pix(f, "color"), [0.5, 0.25, 0.125], atol=1e-7)
        assert pix(f, "final_t") == np.float32(0.125)
        assert pix(f, "contrib") == 3 and pix(f, "term") == 0
        assert pix(f, "depth") == np.float32(0.5 * 1 + 0.25 * 2 + 0.125 * 3)


def serial(alphas):
    """blend_pixel's transmittance recurrence (src/blend.cpp:21-34) on float alphas."""
    t, contrib, term = np.float32(1), 0, 0
    for i, a in enumerate(alphas):
        a = np.float32(a)
        if a < np.float32(1.0) / np.float32(255.0):
            continue
        tmp = t * (np.float32(1) - a)
        if tmp < np.float32(1e-4):
            term = i + 1
            break
        t, contrib = tmp, contrib + 1
    return t, contrib, term


def test_termination_stops_without_commit():
    # alpha 0.99 x 3: T 1 -> 0.01 -> 1e-4 -> the third would go below 1e-4:
    # stop without committing, term = its 1-based list position
    g = np.concatenate([splat(PX + 0.5, PY + 0.5, 1.0, (1, 1, 1), d) for d in (1.0, 2.0, 3.0, 4.0)])
    t = np.float32(1)
    steps = 0
    for _ in range(4):
        tmp = t * (np.float32(1) - np.float32(0.99))
        if tmp < np.float32(1e-4):
            break
        t, steps = tmp, steps + 1
    for f in render_all(g, (0.2, 0.2, 0.2)).values():
        assert pix(f, "contrib") == steps
        assert pix(f, "term") == steps + 1
        assert pix(f, "final_t") == t


def test_skip_below_threshold_counts_in_term():
    # a faint splat (alpha < 1/255) in front is skipped but still counts in
    # the list position; then two opaque ones stop the pixel
    g = np.concatenate([splat(PX + 0.5, PY + 0.5, 0.003, (1, 0, 0), 0.5)] +
                       [splat(PX + 0.5, PY + 0.5, 0.9, (0, 1, 0), d) for d in (1.0, 2.0, 3.0, 4.0, 5.0)])
    t, contrib, term = serial([0.003] + [0.9] * 5)
    assert term > 0 and contrib >= 2
    for f in render_all(g, (0, 0, 0)).values():
        assert pix(f, "contrib") == contrib
        assert pix(f, "term") == term
        assert pix(f, "final_t") == t


def test_gaussianwise_long_list_crosses_groups():
    # 70 faint steps (alpha 0.05) on one pixel: more than two 32-entry groups,
    # so the Gaussian-wise prefix product carries across groups (R5/R6)
    n = 70
    g = np.concatenate([splat(PX + 0.5, PY + 0.5, 0.05, (0.5, 0.25, 1.0), 1.0 + i) for i in range(n)])
    fr = render_all(g, (0.1, 0.2, 0.3))
    t = np.float32(1)
    for _ in range(n):
        t = t * (np.float32(1) - np.float32(0.05))
    for f in fr.values():
        assert pix(f, "contrib") == n and pix(f, "term") == 0
        assert pix(f, "final_t") == t


def test_empty_pixel_is_background():
    g = splat(PX + 0.5, PY + 0.5, 0.5, (1, 0, 0), 1.0)
    for f in render_all(g, (0.25, 0.5, 0.75)).values():
        far = f["color"].reshape(H, W, 3)[0, W - 1]
        assert np.array_equal(far, np.array([0.25, 0.5, 0.75], np.float32))
        assert f["final_t"].reshape(H, W)[0, W - 1] == 1 and f["contrib"].reshape(H, W)[0, W - 1] == 0
