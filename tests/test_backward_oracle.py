"""SURVEY 8f(4) backward render: the oracle's analytic gradient
(oracle/oracle.cpp render_backward) against central finite differences of
the oracle forward (render_reference semantics, src/blend.cpp:8-42) — the
backward is not in the reference, so finite differences of the reference's
own forward are what pin it.  CPU only."""
import numpy as np
import pytest

import oracle_lib as O


def _scene(seed, n=24, W=48, H=40, f=48.0):
    cam = O.make_camera(focal=(f, f), width=W, height=H)
    g3d = O.gen_clustered_scene(n, cam, seed=seed, sigma=0.08, bgfrac=0.5)
    g2d = O.project_all(g3d, cam)
    return g2d, W, H


def _loss(g2d, pl, rg, W, H, pw, ph, bg, dC, dA, dD):
    out = O.render(0, pl, rg, g2d, W, H, pw, ph, bg, lazy=True, threads=1)
    L = (np.dot(out["color"].astype(np.float64), dC) + np.dot(out["alpha"].astype(np.float64), dA)
         + np.dot(out["depth"].astype(np.float64), dD))
    return L, out


FIELD_OF = {"x": ("x", None), "y": ("y", None), "conic_a": ("conic_a", None), "conic_b": ("conic_b", None),
            "conic_c": ("conic_c", None), "opacity": ("opacity", None), "r": ("color", 0), "g": ("color", 1),
            "b": ("color", 2), "depth": ("depth", None)}


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_backward_matches_finite_differences(seed):
    g2d, W, H = _scene(seed)
    pw = ph = 16
    pl, rg = O.bin_tiles(g2d, W, H, pw, ph)
    rng = np.random.default_rng(seed)
    P = W * H
    dC = rng.normal(size=3 * P)
    dA = rng.normal(size=P)
    dD = rng.normal(size=P) * 0.1
    bg = (0.1, 0.2, 0.3)
    G = O.render_backward(pl, rg, g2d, W, H, pw, ph, bg, dC, dA, dD)
    _, base = _loss(g2d, pl, rg, W, H, pw, ph, bg, dC, dA, dD)
    checked = bad = 0
    for i in range(len(g2d)):
        for j, name in enumerate(O.GRAD_FIELDS):
            field, comp = FIELD_OF[name]
            v0 = float(g2d[field][i] if comp is None else g2d[field][i][comp])
            h = max(1e-3 * abs(v0), 1e-3) if name not in ("x", "y") else 2e-3
            vals = []
            same = True
            for sgn in (1, -1):
                g = g2d.copy()
                if comp is None:
                    g[field][i] = np.float32(v0 + sgn * h)
                else:
                    g[field][i][comp] = np.float32(v0 + sgn * h)
                L, out = _loss(g, pl, rg, W, H, pw, ph, bg, dC, dA, dD)
                same &= np.array_equal(out["contrib"], base["contrib"]) and np.array_equal(out["term"], base["term"])
                vals.append(L)
            if not same:
                continue  # a skip / stop decision flipped: not differentiable there
            fd = (vals[0] - vals[1]) / (2 * h)
            checked += 1
            if abs(fd - G[i, j]) > 5e-3 * max(1.0, abs(G[i, j])):
                bad += 1
    assert checked > 150
    assert bad <= checked // 100, (bad, checked)


def test_backward_zero_when_nothing_commits():
    g2d, W, H = _scene(4)
    pl, rg = O.bin_tiles(g2d, W, H, 16, 16)
    P = W * H
    G = O.render_backward(pl, rg, g2d, W, H, 16, 16, (0, 0, 0), np.zeros(3 * P), np.zeros(P), np.zeros(P))
    assert not G.any()
    # an empty list: no splat gets a gradient
    G = O.render_backward(np.zeros(0, np.uint32), np.zeros_like(rg), g2d, W, H, 16, 16, (0, 0, 0),
                          np.ones(3 * P), np.ones(P), np.ones(P))
    assert not G.any()
