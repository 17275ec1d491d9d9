"""CPU: the oracle restatement (oracle/) against the REFERENCE ITSELF
(oracle/_ref: /root/reference/proj/core's unmodified sources built against the
Eigen-subset shim), on the same inputs, bit for bit.

This is what pins the parity chain: GPU == oracle (tests/test_gpu_*.py) and
oracle == reference (here), on the golden fixtures, the C1 frame and C2-scale
scenes, the SPEC known-answer tests and the host bookkeeping (trace counters,
task specs, artifact writers, scene JSON).  The one piece of arithmetic the
reference does NOT own is Eigen's fixed-size evaluation order; the shim
implements Eigen 3.4's x86-64 SSE2 order (oracle/ref_shim/Eigen/Core) — the
same order the oracle documents, so P1-P3 agreement here is conditional on it.
"""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

import oracle_lib as O
import ref_lib as R

pytestmark = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built and /root/reference absent")

HERE = os.path.dirname(os.path.abspath(__file__))
PLANES = ("color", "alpha", "depth", "final_t", "contrib", "term")


def _scene(n, W, H, f, bgfrac=0.12, seed=42, sigma=0.035):
    cam = O.make_camera(focal=(f, f), width=W, height=H)
    return cam, O.gen_clustered_scene(n, cam, seed=seed, sigma=sigma, bgfrac=bgfrac)


@pytest.mark.parametrize("n,W,H,f,bgf,seed", [(10000, 256, 256, 256.0, 1.0, 42), (50000, 1920, 1080, 1000.0, 0.12, 42),
                                              (3000, 640, 480, 500.0, 0.05, 7)])
def test_scene_generator_matches_reference(n, W, H, f, bgf, seed):
    cam = O.make_camera(focal=(f, f), width=W, height=H)
    a = O.gen_clustered_scene(n, cam, seed=seed, bgfrac=bgf)
    b = R.gen_clustered_scene(n, cam, seed=seed, bgfrac=bgf)
    assert a.tobytes() == b.tobytes()


def test_covariance_and_projection_kats_match_reference():
    cam, g3d = _scene(4000, 320, 240, 300.0, bgfrac=0.5)
    for g in g3d[:500]:
        a = np.zeros(9, np.float32)
        b = np.zeros(9, np.float32)
        O.lib().orc_covariance_of(O.p(g.reshape(1)), O.p(a))
        R.lib().ref_covariance_of(O.p(g.reshape(1)), O.p(b))
        assert a.tobytes() == b.tobytes()
    rng = np.random.default_rng(3)
    for _ in range(200):
        jac, Rm, S = rng.normal(size=6), rng.normal(size=9), rng.normal(size=9)
        oa, ob = np.zeros(4), np.zeros(4)
        O.lib().orc_project_covariance(O.p(jac), O.p(Rm), O.p(S), O.p(oa))
        R.lib().ref_project_covariance(O.p(jac), O.p(Rm), O.p(S), O.p(ob))
        assert oa.tobytes() == ob.tobytes()


@pytest.mark.parametrize("n,W,H,f,bgf", [(10000, 256, 256, 256.0, 1.0), (1_000_000, 1920, 1080, 1000.0, 0.12)])
def test_project_all_matches_reference(n, W, H, f, bgf):
    """C1 and the full C2 scene (1M Gaussians): every Gaussian2D byte."""
    cam, g3d = _scene(n, W, H, f, bgfrac=bgf)
    g3d["mean"][::97, 2] = 0.004  # near-plane culls through the input
    a = O.project_all(g3d, cam)
    b = R.project_all(g3d, cam, threads=os.cpu_count() or 1)
    assert len(a) == len(b) and a.tobytes() == b.tobytes()


def test_project_all_rotated_views_match_reference():
    """C5-style yawed views (orthonormal rotation + translation)."""
    cam, g3d = _scene(20000, 960, 540, 500.0)
    for deg in (-15.0, 3.7, 15.0):
        th = np.deg2rad(deg)
        V = np.eye(4, dtype=np.float32)
        V[0, 0], V[0, 2], V[2, 0], V[2, 2] = np.cos(th), np.sin(th), -np.sin(th), np.cos(th)
        V[:3, 3] = (0.3, -0.1, 0.5)
        c = O.make_camera(view=V, focal=(500.0, 500.0), width=960, height=540)
        assert O.project_all(g3d, c).tobytes() == R.project_all(g3d, c).tobytes()


@pytest.mark.parametrize("n,W,H,f,bgf,pw,ph", [(10000, 256, 256, 256.0, 1.0, 16, 16),
                                               (200_000, 1920, 1080, 1000.0, 0.12, 16, 16),
                                               (6000, 250, 130, 250.0, 0.3, 16, 8),
                                               (3000, 100, 60, 100.0, 0.3, 32, 32)])
def test_bin_tiles_and_histogram_match_reference(n, W, H, f, bgf, pw, ph):
    cam, g3d = _scene(n, W, H, f, bgfrac=bgf)
    g2d = O.project_all(g3d, cam)
    pl_a, rg_a = O.bin_tiles(g2d, W, H, pw, ph)
    pl_b, rg_b = R.bin_tiles(g2d, W, H, pw, ph)
    assert np.array_equal(pl_a, pl_b) and np.array_equal(rg_a, rg_b)
    cols, rows = (W + pw - 1) // pw, (H + ph - 1) // ph
    ha, hb = O.tile_load_histogram(rg_a, cols, rows), R.tile_load_histogram(rg_a, cols, rows)
    assert np.array_equal(ha["counts"], hb["counts"])
    assert all(ha[k] == hb[k] for k in ("min", "max", "mean", "p50", "p99"))


@pytest.mark.parametrize("variant", range(5))
def test_c1_frame_all_variants_match_reference(variant):
    """C1 full frame (10k uniform, 256x256): the oracle's render of every
    variant == the reference's run_kernel, every plane bit for bit."""
    cam, g3d = _scene(10000, 256, 256, 256.0, bgfrac=1.0)
    g2d = O.project_all(g3d, cam)
    pl, rg = O.bin_tiles(g2d, 256, 256, 16, 16)
    bg = (0.1, 0.2, 0.3)
    a = O.render(variant, pl, rg, g2d, 256, 256, 16, 16, bg, lazy=False, threads=0)
    b = R.run_kernel(variant, pl, rg, g2d, 256, 256, 16, 16, bg)
    for k in PLANES:
        assert a[k].tobytes() == b[k].tobytes(), k


def test_lazy_oracle_and_threaded_reference_match():
    """The oracle's lazy evaluation (stops evaluating alpha past a pixel's
    term) and the reference's tile-parallel run_kernel wrapper both equal one
    plain reference run_kernel call."""
    cam, g3d = _scene(6000, 192, 128, 192.0)
    g2d = O.project_all(g3d, cam)
    pl, rg = O.bin_tiles(g2d, 192, 128, 16, 8)
    for v in (0, 3):
        one = R.run_kernel(v, pl, rg, g2d, 192, 128, 16, 8, (0.1, 0.2, 0.3), threads=1)
        par = R.run_kernel(v, pl, rg, g2d, 192, 128, 16, 8, (0.1, 0.2, 0.3), threads=4)
        lazy = O.render(v, pl, rg, g2d, 192, 128, 16, 8, (0.1, 0.2, 0.3), lazy=True, threads=0)
        for k in PLANES:
            assert one[k].tobytes() == par[k].tobytes() == lazy[k].tobytes(), (v, k)


def test_golden_digests_are_the_reference_s():
    """The frozen fixture digests (tests/golden/digests.json, written from the
    oracle) are reproduced by the reference's own code."""
    from golden.gen_golden import FIXTURES
    with open(os.path.join(HERE, "golden", "digests.json")) as f:
        frozen = json.load(f)
    for name, (n, W, H, f_, bgf, pw, ph, bg) in FIXTURES.items():
        cam = O.make_camera(focal=(f_, f_), width=W, height=H)
        g3d = R.gen_clustered_scene(n, cam, bgfrac=bgf)
        g2d = R.project_all(g3d, cam)
        pl, rg = R.bin_tiles(g2d, W, H, pw, ph)
        d = frozen[name]
        assert (len(g2d), len(pl)) == (d["n_visible"], d["K"])
        assert [R.fnv1a64(x) for x in (g3d, g2d, pl, rg)] == [d["g3d"], d["g2d"], d["point_list"], d["tile_ranges"]]
        for v, tag in ((0, "render_reference"), (2, "render_gaussianwise")):
            r = R.run_kernel(v, pl, rg, g2d, W, H, pw, ph, bg)
            assert {k: R.fnv1a64(r[k]) for k in PLANES} == d[tag], (name, tag)


def test_blend_kats_match_reference():
    """SPEC blend KATs and 2,000 random step lists (acceptance #9 style)."""
    cases = [([0.5, 0.5, 0.5], [[1, 0, 0], [0, 1, 0], [0, 0, 1]]), ([0.999, 0.999], None), ([], None),
             ([0.001, 0.5, 0.99, 0.99, 0.99], None)]
    rng = np.random.default_rng(9)
    for _ in range(2000):
        k = int(rng.integers(0, 80))
        a = rng.choice([0.0, 0.001, 0.004, 0.2, 0.6, 0.99], size=k) * rng.uniform(0.5, 1.0, size=k)
        cases.append((np.minimum(a, 0.99), rng.uniform(0, 1, size=(k, 3))))
    for alphas, cols in cases:
        a = np.asarray(alphas, np.float32)
        dep = np.linspace(1, 2, len(a)).astype(np.float32)
        o = O.blend_pixel(a, cols, dep, bg=(0.1, 0.2, 0.3))
        r = R.blend_pixel(a, cols, dep, bg=(0.1, 0.2, 0.3))
        assert o["color"].tobytes() == r["color"].tobytes()
        assert (o["alpha"], o["depth"], o["final_t"], o["contrib"], o["term"]) == \
               (r["alpha"], r["depth"], r["final_t"], r["contrib"], r["term"])
        assert O.lib().orc_termination_index(O.p(a), len(a)) == R.lib().ref_termination_index(O.p(a), len(a))


def test_eval_alpha_and_prefix_product_match_reference():
    cam, g3d = _scene(2000, 128, 128, 128.0, bgfrac=0.5)
    g2d = O.project_all(g3d, cam)
    rng = np.random.default_rng(5)
    import ctypes as C
    for g in g2d[:300]:
        for _ in range(8):
            px, py = (np.float32(v) for v in rng.uniform(0, 128, 2))
            pa, aa, pb, ab = C.c_float(), C.c_float(), C.c_float(), C.c_float()
            O.lib().orc_eval_alpha(O.p(g.reshape(1)), px, py, C.byref(pa), C.byref(aa))
            R.lib().ref_eval_alpha(O.p(g.reshape(1)), px, py, C.byref(pb), C.byref(ab))
            assert (pa.value, aa.value) == (pb.value, ab.value)
    for _ in range(200):
        f = rng.uniform(0.9, 1.0, 32).astype(np.float32)
        oa, ob = np.zeros(32, np.float32), np.zeros(32, np.float32)
        ta, tb = C.c_float(), C.c_float()
        O.lib().orc_warp_prefix_product_f32(O.p(f), np.float32(0.7), O.p(oa), C.byref(ta))
        R.lib().ref_warp_prefix_product_f32(O.p(f), np.float32(0.7), O.p(ob), C.byref(tb))
        assert oa.tobytes() == ob.tobytes() and ta.value == tb.value
