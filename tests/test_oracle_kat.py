"""CPU: pin the oracle against every SPEC.md known-answer test for the hot path
 and the reference's stated properties.  No GPU needed."""
from __future__ import annotations

import ctypes as C
import math

import numpy as np
import pytest

import oracle_lib as O

L = O.lib()


def g3d(mean=(0, 0, 10), scale=(1, 1, 1), rot=(1, 0, 0, 0), opacity=1.0, color=(0, 0, 0)):
    g = np.zeros(1, dtype=O.G3D_DTYPE)
    g["mean"], g["scale"], g["rot"], g["opacity"], g["color"] = mean, scale, rot, opacity, color
    return g


def cov(g):
    out = np.zeros(9, np.float32)
    L.orc_covariance_of(O.p(g), O.p(out))
    return out.reshape(3, 3)


# ---- covariance_of ----
def test_covariance_identity():
    assert np.array_equal(cov(g3d()), np.eye(3, dtype=np.float32))


def test_covariance_diagonal():
    assert np.array_equal(cov(g3d(scale=(2, 1, 1))), np.diag([4, 1, 1]).astype(np.float32))


def test_covariance_rotated_90_about_z():
    h = math.sqrt(0.5)
    c = cov(g3d(scale=(2, 1, 1), rot=(h, 0, 0, h)))
    assert np.allclose(c, np.diag([1, 4, 1]), atol=1e-6)


def test_covariance_spd_random():
    rng = np.random.default_rng(0)
    for _ in range(1000):
        q = rng.normal(size=4)
        q /= np.linalg.norm(q)
        c = cov(g3d(scale=rng.uniform(0.01, 2, 3), rot=q)).astype(np.float64)
        assert np.allclose(c, c.T, atol=0) and np.linalg.eigvalsh(c).min() > 0


# ---- project_covariance / project_gaussian ----
def test_project_covariance_identity():
    jac = np.array([1, 0, 0, 0, 1, 0], np.float64)
    out = np.zeros(4)
    L.orc_project_covariance(O.p(jac), O.p(np.eye(3).reshape(-1).copy()), O.p(np.eye(3).reshape(-1).copy()), O.p(out))
    assert np.array_equal(out, [1, 0, 0, 1])


def test_project_gaussian_pinhole_kat():
    cam = O.make_camera(focal=(100, 100), width=0, height=0)
    out = np.zeros(1, O.G2D_DTYPE)
    assert L.orc_project_gaussian(O.p(g3d(mean=(0, 0, 10))), C.byref(cam), O.p(out)) == 1
    o = out[0]
    assert o["conic_a"] == np.float32(0.01) and o["conic_b"] == 0 and o["conic_c"] == np.float32(0.01)
    assert o["radius"] == 30.0 and o["depth"] == 10.0 and o["x"] == 0 and o["y"] == 0


def test_project_gaussian_near_cull():
    cam = O.make_camera(focal=(100, 100), width=64, height=64)
    out = np.zeros(1, O.G2D_DTYPE)
    for z in (0.01, 0.005, -3.0):
        assert L.orc_project_gaussian(O.p(g3d(mean=(0, 0, z))), C.byref(cam), O.p(out)) == 0


def test_project_all_preserves_order():
    cam = O.make_camera(focal=(100, 100), width=64, height=64)
    gs = np.concatenate([g3d(mean=(0, 0, z)) for z in (5, 0.001, 7, 9, -1, 3)])
    out = O.project_all(gs, cam)
    assert list(out["depth"]) == [5, 7, 9, 3]


# ---- bin_tiles ----
def test_bin_empty():
    pl, rg = O.bin_tiles(np.zeros(0, O.G2D_DTYPE), 64, 64, 16, 16)
    assert len(pl) == 0 and not rg.any() and len(rg) == 32


def test_bin_grid_960x540_16x8():
    pl, rg = O.bin_tiles(np.zeros(0, O.G2D_DTYPE), 960, 540, 16, 8)
    assert len(rg) == 2 * 4080


def test_bin_single_contained():
    g = np.zeros(1, O.G2D_DTYPE)
    g["x"], g["y"], g["radius"], g["depth"] = 24.0, 40.0, 3.0, 1.0
    pl, rg = O.bin_tiles(g, 64, 64, 16, 16)
    assert list(pl) == [0]
    t = 2 * 4 + 1
    assert rg[2 * t] == 0 and rg[2 * t + 1] == 1


def _scene(n, W, H, f, seed, bgf=0.5):
    cam = O.make_camera(focal=(f, f), width=W, height=H)
    return O.project_all(O.gen_clustered_scene(n, cam, seed=seed, bgfrac=bgf), cam)


def test_bin_partition_sort_conservative():
    W = H = 64
    for seed in range(5):
        g2 = _scene(200, W, H, 64.0, seed)
        pl, rg = O.bin_tiles(g2, W, H, 16, 16)
        starts, ends = rg[0::2], rg[1::2]
        assert starts[0] == 0 and ends[-1] == len(pl) and np.array_equal(starts[1:], ends[:-1])
        for t in range(16):
            ids = pl[starts[t]:ends[t]]
            key = list(zip(g2["depth"][ids], ids))
            assert key == sorted(key)
        # conservativeness: alpha >= 1/255 at a pixel of tile t => listed in t
        for t in range(16):
            tx, ty = t % 4, t // 4
            listed = set(pl[starts[t]:ends[t]].tolist())
            for i in range(len(g2)):
                if i in listed:
                    continue
                for py in range(ty * 16, ty * 16 + 16, 5):
                    for px in range(tx * 16, tx * 16 + 16, 5):
                        pw_, al = C.c_float(), C.c_float()
                        L.orc_eval_alpha(O.p(g2[i:i + 1]), px + 0.5, py + 0.5, C.byref(pw_), C.byref(al))
                        assert al.value < 1 / 255 or pw_.value > 0


# ---- tile_load_histogram ----
def test_histogram_kats():
    rg = np.array([0, 1, 1, 3, 3, 6], np.uint32)
    h = O.tile_load_histogram(rg, 3, 1)
    assert h["mean"] == 2.0 and h["max"] == 3 and h["min"] == 1 and h["p50"] == 2 and h["p99"] == 3
    h0 = O.tile_load_histogram(np.zeros(8, np.uint32), 2, 2)
    assert h0["max"] == 0


# ---- eval_alpha ----
def test_eval_alpha_kats():
    g = np.zeros(1, O.G2D_DTYPE)
    g["conic_a"], g["conic_c"], g["opacity"] = 1, 1, 0.5
    pw_, al = C.c_float(), C.c_float()
    L.orc_eval_alpha(O.p(g), 0.0, 0.0, C.byref(pw_), C.byref(al))
    assert pw_.value == 0 and al.value == np.float32(0.5)
    g["opacity"] = 1.0
    L.orc_eval_alpha(O.p(g), 2.0, 0.0, C.byref(pw_), C.byref(al))
    assert pw_.value == -2.0 and abs(al.value - math.exp(-2)) < 1e-7
    L.orc_eval_alpha(O.p(g), 0.0, 0.0, C.byref(pw_), C.byref(al))
    assert al.value == np.float32(0.99)


# ---- blend_pixel / termination_index ----
def test_blend_empty():
    r = O.blend_pixel([], bg=(0.1, 0.2, 0.3))
    assert np.allclose(r["color"], [0.1, 0.2, 0.3]) and r["alpha"] == 0 and r["final_t"] == 1 and r["contrib"] == 0


@pytest.mark.parametrize("gw", [False, True])
def test_blend_three_half(gw):
    r = O.blend_pixel([0.5] * 3, colors=np.eye(3), depths=[1, 2, 3], gaussianwise=gw)
    assert np.allclose(r["color"], [0.5, 0.25, 0.125], atol=1e-6)
    assert r["final_t"] == 0.125 and r["contrib"] == 3 and r["term"] == 0


def test_blend_two_0999():
    r = O.blend_pixel([0.999, 0.999])
    assert r["contrib"] == 1 and r["term"] == 2 and abs(r["final_t"] - 0.001) < 1e-6


def test_termination_index():
    a = np.array([0.001, 0.002], np.float32)
    assert L.orc_termination_index(O.p(a), 2) == 0
    a = np.array([0.99999], np.float32)
    assert L.orc_termination_index(O.p(a), 1) == 1
    a = np.array([0.999, 0.999], np.float32)
    assert L.orc_termination_index(O.p(a), 2) == 2


def test_blend_invariants_random_lists():
    rng = np.random.default_rng(1)
    for _ in range(2000):
        n = int(rng.integers(0, 60))
        al = rng.uniform(0, 0.99, n).astype(np.float32) * (rng.uniform(size=n) < 0.7)
        term = L.orc_termination_index(O.p(al) if n else None, n)
        # sentinel colour after term must never show up
        cols = np.zeros((n, 3), np.float32)
        if term:
            cols[term - 1:] = 1000.0
        r = O.blend_pixel(al, colors=cols)
        assert r["final_t"] <= 1.0 and r["alpha"] + r["final_t"] == np.float32(1.0) or \
            np.float32(1.0) - r["final_t"] == r["alpha"]
        assert r["term"] == term
        assert (r["color"] < 1.0).all()


# ---- warp_prefix_product ----
def test_prefix_product_kats():
    out = np.zeros(32, np.float32)
    to = C.c_float()
    L.orc_warp_prefix_product_f32(O.p(np.ones(32, np.float32)), 0.7, O.p(out), C.byref(to))
    assert (out == np.float32(0.7)).all() and to.value == np.float32(0.7)
    L.orc_warp_prefix_product_f32(O.p(np.full(32, 0.5, np.float32)), 1.0, O.p(out), C.byref(to))
    assert np.array_equal(out, (0.5 ** np.arange(1, 33)).astype(np.float32))


def test_prefix_product_vs_serial_double():
    rng = np.random.default_rng(2)
    out = np.zeros(32)
    to = C.c_double()
    for _ in range(1000):
        f = rng.uniform(0.9, 1.0, 32)
        L.orc_warp_prefix_product_f64(O.p(f), 1.0, O.p(out), C.byref(to))
        assert np.max(np.abs(out - np.cumprod(f)) / np.cumprod(f)) < 1e-12


# ---- variants agree, warp step counts ----
def test_variants_match_reference_random_scenes():
    for seed in range(12):
        W = H = 128
        g2 = _scene(int(200 + 300 * seed), W, H, 128.0, seed, bgf=0.3)
        pl, rg = O.bin_tiles(g2, W, H, 16, 16)
        ref = O.render(0, pl, rg, g2, W, H, 16, 16, (0.1, 0.2, 0.3), lazy=False, threads=1)
        for v in range(1, 5):
            got = O.render(v, pl, rg, g2, W, H, 16, 16, (0.1, 0.2, 0.3), lazy=True, threads=4)
            assert np.array_equal(got["contrib"], ref["contrib"]) and np.array_equal(got["term"], ref["term"])
            for k in ("color", "alpha", "depth"):
                rel = np.abs(got[k] - ref[k]) / np.maximum(1, np.abs(ref[k]))
                assert rel.max() <= 1e-5
            if v in (1, 4):
                assert all(np.array_equal(got[k], ref[k]) for k in ref)


def test_warp_steps():
    t = np.ones(32, np.int64)
    assert L.orc_warp_steps_pixelwise(O.p(t), 32, 5000) == 1
    t = np.zeros(32, np.int64)
    t[:3] = [10, 20, 1000]
    assert L.orc_warp_steps_pixelwise(O.p(t), 32, 5000) == 5000
    assert L.orc_warp_steps_gaussianwise(1, 100) == 1
    assert L.orc_warp_steps_gaussianwise(33, 100) == 2
    assert L.orc_warp_steps_gaussianwise(0, 1000) == 32


# ---- third-party pin: glibc expf (the reference's std::exp(float)) ----
def test_expf_restatement_exhaustive():
    bad = np.zeros(8, np.float32)
    n = L.orc_expf_exhaustive_check(np.float32(-103.9), np.float32(0.0), O.p(bad), 8)
    # glibc 2.39 special-cases one input in this range; the GPU path reproduces it
    assert n == 1 and bad[0] == np.float32(float.fromhex("-0x1.f8cbb2p+5"))


def test_lazy_equals_faithful():
    W = H = 96
    g2 = _scene(3000, W, H, 96.0, 7, bgf=0.2)
    pl, rg = O.bin_tiles(g2, W, H, 16, 16)
    for v in (0, 2):
        a = O.render(v, pl, rg, g2, W, H, 16, 16, (0, 0, 0), lazy=False, threads=1)
        b = O.render(v, pl, rg, g2, W, H, 16, 16, (0, 0, 0), lazy=True, threads=3)
        assert all(np.array_equal(a[k], b[k]) for k in a)
