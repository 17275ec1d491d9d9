"""GPU parity: every CUDA stage vs the CPU oracle, through the C-ABI.

Bars (SURVEY §8.0 / BASELINE north star):
  * preprocess, binning, tile stats: bit-exact;
  * BS_ALPHA_EXACT render: pixel-wise variants bit-exact on every plane;
    Gaussian-wise variants bit-exact on alpha / final_t / contrib / term and
    colour/depth within 1e-6 abs (double-sum association only);
  * BS_ALPHA_FAST render: RGB and T within 1e-4 abs on pixels whose
    contrib/term match; mismatching pixels are counted and must stay rare.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

import oracle_lib as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_2412_17378_b200 import _native as N  # noqa: E402
from paper_2412_17378_b200 import api  # noqa: E402
from paper_2412_17378_b200 import sharding  # noqa: E402

DEV = "cuda"
PLANES_F = ("color", "alpha", "depth", "final_t")


def ncam(o_cam: O.Camera) -> N.Camera:
    return N.Camera.from_buffer_copy(bytes(o_cam))


def scene(n, W, H, f, bgfrac=0.12, seed=42, sigma=0.035):
    cam = O.make_camera(focal=(f, f), width=W, height=H)
    return O.gen_clustered_scene(n, cam, seed=seed, sigma=sigma, bgfrac=bgfrac), cam


def to_dev_splats(g2d: np.ndarray) -> api.DeviceSplats:
    return api.splats_from_g2d(g2d, DEV)


# ---------------------------------------------------------------------------
def test_library_loads_and_device():
    assert N.lib().bs_abi_version() == 1
    assert api.sm_count() >= 1


def test_exact_expf_matches_libm():
    """The render's own exp (glibc_expf_fast through the shared-memory table,
    as eval_step calls it) on EVERY float of its input range
    [-0x1.9fe368p6, 0] (~1.12e9 values, +0 and -0 included) against the host
    libm expf the reference calls (src/blend.cpp:12): bit for bit."""
    lo_bits = int(np.float32(float.fromhex("-0x1.9fe368p6")).view(np.uint32))
    first, last = 0x80000000, lo_bits  # -0.0 .. -103.97 (negative floats grow in bits)
    chunk = 1 << 27
    y = torch.empty(chunk, dtype=torch.float32, device=DEV)
    yh = torch.empty(chunk, dtype=torch.float32, pin_memory=True)
    bad = total = 0
    b = first
    while b <= last:
        n = min(chunk, last - b + 1)
        N.call("bs_test_expf_range", b, n, y.data_ptr(), N.ALPHA_EXACT, api._stream(DEV))
        yh[:n].copy_(y[:n])
        bad += O.lib().orc_expf_compare_range(b, n, yh.data_ptr())
        total += n
        b += n
    N.call("bs_test_expf_range", 0, 1, y.data_ptr(), N.ALPHA_EXACT, api._stream(DEV))  # +0.0
    yh[:1].copy_(y[:1])
    bad += O.lib().orc_expf_compare_range(0, 1, yh.data_ptr())
    assert total == last - first + 1 > 1_100_000_000
    assert bad == 0
    # the array form on a few values outside the render's range (general path)
    x = np.array([float.fromhex("-0x1.f8cbb2p+5"), -50.0, -103.0, -104.5, 1.5, 80.0], np.float32)
    xd = torch.from_numpy(x).to(DEV)
    yd = torch.empty_like(xd)
    N.call("bs_test_expf", xd.data_ptr(), yd.data_ptr(), x.size, N.ALPHA_EXACT, api._stream(DEV))
    assert O.lib().orc_expf_compare_batch(O.p(x), O.p(yd.cpu().numpy()), x.size) == 0


def test_preprocess_bit_exact():
    g3d, cam = scene(20000, 256, 256, 256.0, bgfrac=0.5)
    ref = O.project_all(g3d, cam)
    d = api.g3d_to_device(g3d)
    s = api.project_all(d, len(g3d), ncam(cam))
    got = api.splats_to_g2d(s)
    assert len(got) == len(ref)
    assert got.tobytes() == ref.tobytes()


def test_preprocess_culls_and_empty():
    cam = O.make_camera(focal=(100, 100), width=64, height=64)
    g = np.zeros(3, dtype=O.G3D_DTYPE)
    g["scale"] = 1.0
    g["rot"][:, 0] = 1.0
    g["opacity"] = 0.5
    g["mean"][0] = (0, 0, 0.005)   # behind the near plane
    g["mean"][1] = (0, 0, 10.0)
    g["mean"][2] = (1, -1, 5.0)
    ref = O.project_all(g, cam)
    s = api.project_all(api.g3d_to_device(g), 3, ncam(cam))
    got = api.splats_to_g2d(s)
    assert got.tobytes() == ref.tobytes() and len(got) == 2
    s0 = api.project_all(torch.empty(56, dtype=torch.uint8, device=DEV), 0, ncam(cam))
    assert int(s0.n_visible.item()) == 0


@pytest.mark.parametrize("W,H,pw,ph,n", [(256, 256, 16, 16, 10000), (250, 130, 16, 8, 4000), (960, 540, 16, 8, 30000),
                                         (64, 64, 16, 16, 1), (100, 60, 32, 32, 3000)])
def test_binning_bit_exact(W, H, pw, ph, n):
    g3d, cam = scene(n, W, H, float(W), bgfrac=0.3)
    g2d = O.project_all(g3d, cam)
    pl_ref, rg_ref = O.bin_tiles(g2d, W, H, pw, ph)
    s = to_dev_splats(g2d)
    b = api.bin_tiles(s, W, H, pw, ph)
    assert b.k == len(pl_ref)
    assert np.array_equal(b.tile_ranges.cpu().numpy().view(np.uint32), rg_ref)
    assert np.array_equal(b.point_list.cpu().numpy().view(np.uint32), pl_ref)


@pytest.mark.parametrize("W,H,f,n,bgfrac", [(1920, 1080, 1000.0, 200_000, 0.12),   # ~600 chunks
                                             (3840, 2160, 2000.0, 60_000, 0.12),    # C4 grid: 32,400 tiles
                                             (8192, 4096, 4096.0, 3000, 1.0)])      # 131,072 tiles: radix fallback
def test_binning_bit_exact_large(W, H, f, n, bgfrac):
    """Chunked counting scatter at full 1080p / 4K grids (many chunks, splats
    straddling chunk bounds) and the radix fallback beyond its smem limit."""
    g3d, cam = scene(n, W, H, f, bgfrac=bgfrac)
    g2d = O.project_all(g3d, cam)
    pl_ref, rg_ref = O.bin_tiles(g2d, W, H, 16, 16)
    b = api.bin_tiles(to_dev_splats(g2d), W, H, 16, 16)
    assert b.k == len(pl_ref)
    assert np.array_equal(b.tile_ranges.cpu().numpy().view(np.uint32), rg_ref)
    assert np.array_equal(b.point_list.cpu().numpy().view(np.uint32), pl_ref)


@pytest.mark.parametrize("W,H,f,n,bgfrac,misaligned", [(960, 540, 500.0, 30000, 0.3, False),
                                                        (1920, 1080, 1000.0, 40000, 0.12, False),
                                                        (960, 540, 500.0, 30001, 0.3, True)])
def test_fused_project_bin_matches_reference(W, H, f, n, bgfrac, misaligned):
    """bs_preprocess_bin_count (the frame pipeline's projection fused with the
    per-splat binning pass, splats left uncompacted) + bs_bin_sort: the
    visible splats equal project_all's, and mapping every list entry through
    the compaction gives bin_tiles' point_list and ranges exactly.
    misaligned: the scene pointer only 8-byte aligned (the kernel then skips
    its 16-byte cp.async staging)."""
    g3d, cam = scene(n, W, H, f, bgfrac=bgfrac)
    g3d["mean"][::53, 2] = 0.004  # near-plane culls scattered through the input
    g2d = O.project_all(g3d, cam)
    pl_ref, rg_ref = O.bin_tiles(g2d, W, H, 16, 16)
    vis = np.array([len(O.project_all(g3d[i:i + 1], cam)) == 1 for i in range(n)])
    assert vis.sum() == len(g2d) < n
    d = api.g3d_to_device(g3d)
    if misaligned:
        buf = torch.zeros(d.numel() + 16, dtype=torch.uint8, device=DEV)
        buf[8:8 + d.numel()] = d
        d = buf[8:8 + d.numel()]
        assert d.data_ptr() % 16 == 8
    s = api.DeviceSplats.empty(n, DEV)
    counts = torch.zeros(2, dtype=torch.int32, device=DEV)
    b = api.Binner(W, H, 16, 16, DEV)
    c = ncam(cam)

    def count():
        N.call("bs_preprocess_bin_count", d.data_ptr(), n, C.byref(c), None, s.c(), counts.data_ptr(), W, H, 16, 16,
               b.k_dev.data_ptr(), b.ws.data_ptr(), b.ws.numel(), api._stream(DEV))

    b._ensure_ws(n, 0)
    count()
    k = b.read_k()
    b._ensure_ws(n, int(k * 1.25) + 1024)
    count()
    assert b.read_k() == k == len(pl_ref)
    pl = torch.empty(max(k, 1), dtype=torch.int32, device=DEV)
    N.call("bs_bin_sort", s.c(), n, counts.data_ptr(), W, H, 16, 16, k, pl.data_ptr(), b.tile_ranges.data_ptr(),
           b.ws.data_ptr(), b.ws.numel(), api._stream(DEV))
    torch.cuda.synchronize()
    cnt = counts.cpu().numpy()
    assert cnt[0] == n and cnt[1] == vis.sum()
    assert np.array_equal(b.tile_ranges.cpu().numpy().view(np.uint32), rg_ref)
    comp = np.cumsum(vis) - 1
    got = pl[:k].cpu().numpy().view(np.uint32)
    assert vis[got].all()
    assert np.array_equal(comp[got].astype(np.uint32), pl_ref)
    idx = torch.from_numpy(np.nonzero(vis)[0]).to(DEV)
    sv = api.DeviceSplats(s.xyab[idx].contiguous(), s.cop[idx].contiguous(), s.rgbr[idx].contiguous(),
                          torch.tensor([len(idx)], dtype=torch.int32, device=DEV))
    assert api.splats_to_g2d(sv).tobytes() == g2d.tobytes()


@pytest.mark.parametrize("W,H,pw,ph,n", [(250, 130, 16, 16, 5000), (960, 540, 16, 16, 60000), (200, 120, 8, 8, 3000),
                                         (300, 170, 16, 8, 8000)])
@pytest.mark.parametrize("variant", [3, 4])
def test_super_tile_lists_render_exact(W, H, pw, ph, n, variant):
    """The frame pipeline's super-tile path through the C-ABI: projection +
    counting at 2pw x 2ph (bs_preprocess_bin_count_super), lists sorted at
    2pw x 2ph, per-tile super ranges, and bs_render_forward_super keeping each
    tile's members — equal to the oracle's render of the pw x ph lists
    (contrib / term / T exact; the pw x ph lengths equal bin_tiles')."""
    g3d, cam = scene(n, W, H, float(W), bgfrac=0.3)
    g2d = O.project_all(g3d, cam)
    pl, rg = O.bin_tiles(g2d, W, H, pw, ph)
    bg = (0.1, 0.2, 0.3)
    ref = O.render(variant, pl, rg, g2d, W, H, pw, ph, bg, lazy=True, threads=0)
    d = api.g3d_to_device(g3d)
    s = api.DeviceSplats.empty(n, DEV)
    counts = torch.zeros(2, dtype=torch.int32, device=DEV)
    b = api.Binner(W, H, 2 * pw, 2 * ph, DEV)
    T = ((W + pw - 1) // pw) * ((H + ph - 1) // ph)
    r16 = torch.empty(2 * T, dtype=torch.int32, device=DEV)
    aux = torch.empty(N.lib().bs_super_aux_bytes(W, H, pw, ph), dtype=torch.uint8, device=DEV)
    c = ncam(cam)
    st = api._stream(DEV)

    def count():
        N.call("bs_preprocess_bin_count_super", d.data_ptr(), n, C.byref(c), None, s.c(), counts.data_ptr(), W, H, pw,
               ph, b.k_dev.data_ptr(), b.ws.data_ptr(), b.ws.numel(), r16.data_ptr(), aux.data_ptr(), aux.numel(), st)

    b._ensure_ws(n, 0)
    count()
    k = b.read_k()
    b._ensure_ws(n, int(k * 1.25) + 1024)
    count()
    pl2 = torch.empty(max(k, 1), dtype=torch.int32, device=DEV)
    N.call("bs_bin_sort", s.c(), n, counts.data_ptr(), W, H, 2 * pw, 2 * ph, k, pl2.data_ptr(),
           b.tile_ranges.data_ptr(), b.ws.data_ptr(), b.ws.numel(), st)
    lens = r16.cpu().numpy().view(np.uint32)
    assert np.array_equal(lens[1::2] - lens[0::2], rg[1::2] - rg[0::2])  # pw x ph list lengths
    rt = torch.empty(2 * T, dtype=torch.int32, device=DEV)
    N.call("bs_super_tile_ranges", b.tile_ranges.data_ptr(), W, H, pw, ph, rt.data_ptr(), st)
    frame = api.DeviceFrame.empty(W, H, DEV)
    ws = torch.zeros(N.lib().bs_render_workspace_bytes(W, H), dtype=torch.uint8, device=DEV)
    bgc = (C.c_float * 3)(*bg)
    N.call("bs_render_forward_super", variant, None, N.ALPHA_EXACT, s.c(), pl2.data_ptr(), rt.data_ptr(), None, W, H,
           pw, ph, bgc, frame.c(), ws.data_ptr(), ws.numel(), st)
    torch.cuda.synchronize()
    got = frame.to_numpy()
    for key in ("contrib", "term"):
        assert np.array_equal(got[key], ref[key]), key
    for key in ("final_t", "alpha"):
        assert np.array_equal(got[key].view(np.uint32), ref[key].view(np.uint32)), key
    if variant == 4:  # SharedMemOpt: serial double sums, bit-exact
        assert np.array_equal(got["color"].view(np.uint32), ref["color"].view(np.uint32))
    else:
        assert np.max(np.abs(got["color"] - ref["color"])) <= 1e-6


@pytest.mark.parametrize("W,H", [(250, 130), (96, 80)])
def test_super_tile_membership_crafted(W, H):
    """bs_render_forward_super on crafted splats: lists binned at 32x32 from
    the same splats (bs_bin_count / bs_bin_sort at 2pw x 2ph), members kept by
    the 16x16 rectangle test — including splats whose rectangle edges sit on
    every parity of the super-tile grid and huge radii (the fast test's
    fallback at ceil(radius) >= 1e9, and edges beyond int range)."""
    rng = np.random.default_rng(7)
    m = 3000
    g = np.zeros(m, dtype=O.G2D_DTYPE)
    g["x"] = rng.uniform(-40, W + 40, m)
    g["y"] = rng.uniform(-40, H + 40, m)
    g["radius"] = np.where(rng.uniform(size=m) < 0.5, rng.integers(1, 40, m) - 0.5, rng.uniform(0.1, 60, m))
    g["radius"][:6] = [1e8, 3e9, 5e10, 2.5e9, 1e12, 7.0]
    g["x"][:6] = [10.0, -1e9, 50.0, W / 2, -3e11, 15.9]
    g["conic_a"] = rng.uniform(0.001, 0.05, m)
    g["conic_c"] = rng.uniform(0.001, 0.05, m)
    g["conic_b"] = rng.uniform(-0.0005, 0.0005, m)
    g["opacity"] = rng.uniform(0.05, 0.9, m)
    g["color"] = rng.uniform(0, 1, (m, 3))
    g["depth"] = rng.uniform(1, 10, m)
    pl, rg = O.bin_tiles(g, W, H, 16, 16)
    bg = (0.1, 0.2, 0.3)
    s = to_dev_splats(g)
    b2 = api.bin_tiles(s, W, H, 32, 32)
    T = ((W + 15) // 16) * ((H + 15) // 16)
    rt = torch.empty(2 * T, dtype=torch.int32, device=DEV)
    st = api._stream(DEV)
    N.call("bs_super_tile_ranges", b2.tile_ranges.data_ptr(), W, H, 16, 16, rt.data_ptr(), st)
    bgc = (C.c_float * 3)(*bg)
    for variant in (3, 4):
        ref = O.render(variant, pl, rg, g, W, H, 16, 16, bg, lazy=True, threads=0)
        frame = api.DeviceFrame.empty(W, H, DEV)
        ws = torch.zeros(N.lib().bs_render_workspace_bytes(W, H), dtype=torch.uint8, device=DEV)
        N.call("bs_render_forward_super", variant, None, N.ALPHA_EXACT, s.c(), b2.point_list.data_ptr(),
               rt.data_ptr(), None, W, H, 16, 16, bgc, frame.c(), ws.data_ptr(), ws.numel(), st)
        torch.cuda.synchronize()
        got = frame.to_numpy()
        for key in ("contrib", "term"):
            assert np.array_equal(got[key], ref[key]), (variant, key)
        assert np.array_equal(got["final_t"].view(np.uint32), ref["final_t"].view(np.uint32)), variant
        assert np.max(np.abs(got["color"] - ref["color"])) <= 1e-6


def test_binning_radix_path_bit_exact():
    """BS_BIN_RADIX=1 (expand + stable tile radix sort) stays bit-exact too."""
    import os
    import subprocess
    import sys
    code = ("import sys; sys.path[:0] = ['tests', '.']; import test_gpu_parity as t; "
            "t.test_binning_bit_exact(960, 540, 16, 8, 30000); t.test_binning_depth_ties_and_empty(); "
            "t.test_binning_bit_exact_large(1920, 1080, 1000.0, 100000, 0.12); print('radix ok')")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=dict(os.environ, BS_BIN_RADIX="1"),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "radix ok" in r.stdout, r.stdout + r.stderr


def test_binning_depth_ties_and_empty():
    # many equal depths: ties must resolve by compacted index
    g2d = np.zeros(500, dtype=O.G2D_DTYPE)
    rng = np.random.default_rng(3)
    g2d["x"] = rng.uniform(-20, 84, 500)
    g2d["y"] = rng.uniform(-20, 84, 500)
    g2d["radius"] = rng.uniform(0, 30, 500)
    g2d["depth"] = rng.choice([1.0, 2.0, 2.5], 500)
    g2d["conic_a"] = g2d["conic_c"] = 1.0
    g2d["opacity"] = 0.5
    pl_ref, rg_ref = O.bin_tiles(g2d, 64, 64, 16, 16)
    b = api.bin_tiles(to_dev_splats(g2d), 64, 64, 16, 16)
    assert np.array_equal(b.point_list.cpu().numpy().view(np.uint32), pl_ref)
    assert np.array_equal(b.tile_ranges.cpu().numpy().view(np.uint32), rg_ref)
    e = api.bin_tiles(to_dev_splats(np.zeros(0, dtype=O.G2D_DTYPE)), 64, 64, 16, 16)
    assert e.k == 0 and not e.tile_ranges.cpu().numpy().any()


@pytest.mark.parametrize("W,H,pw,ph,n", [(960, 540, 16, 8, 30000),      # 4,080 tiles
                                         (1920, 1080, 16, 16, 30000),   # 8,160: single-CTA bitonic path
                                         (3840, 2160, 16, 16, 20000)])  # 32,400: radix path
def test_tile_stats_match_oracle(W, H, pw, ph, n):
    g3d, cam = scene(n, W, H, float(W))
    g2d = O.project_all(g3d, cam)
    pl, rg = O.bin_tiles(g2d, W, H, pw, ph)
    cols, rows = (W + pw - 1) // pw, (H + ph - 1) // ph
    T = cols * rows
    ref = O.tile_load_histogram(rg, cols, rows)
    b = api.bin_tiles(to_dev_splats(g2d), W, H, pw, ph)
    st = api.tile_load_histogram(b)
    s = st.summary()
    for k in ("min", "max", "p50", "p99"):
        assert s[k] == ref[k], k
    assert s["mean"] == ref["mean"]
    assert s["tiles"] == T
    counts = st.counts.cpu().numpy().view(np.uint32)[:T]
    assert np.array_equal(counts, ref["counts"])
    order = st.task_order.cpu().numpy()[:T]
    exp = np.lexsort((np.arange(T), -ref["counts"].astype(np.int64)))
    assert np.array_equal(order, exp)


def _gpu_render(variant, g2d, W, H, pw, ph, bg, mode):
    s = to_dev_splats(g2d)
    b = api.bin_tiles(s, W, H, pw, ph)
    st = api.tile_load_histogram(b)
    f = api.render_forward(variant, s, b, W, H, pw, ph, bg, mode, st.task_order)
    torch.cuda.synchronize()
    return f.to_numpy(), b


def _oracle_render(variant, g2d, W, H, pw, ph, bg):
    pl, rg = O.bin_tiles(g2d, W, H, pw, ph)
    return O.render(variant, pl, rg, g2d, W, H, pw, ph, bg, lazy=True, threads=0)


CASES = [(256, 256, 16, 16, 10000, 1.0), (192, 128, 16, 8, 6000, 0.12), (250, 130, 16, 16, 5000, 0.3),
         (100, 60, 32, 32, 3000, 0.3), (90, 70, 8, 8, 2000, 0.3)]


@pytest.mark.parametrize("W,H,pw,ph,n,bgfrac", CASES)
@pytest.mark.parametrize("variant", range(5))
def test_render_exact(variant, W, H, pw, ph, n, bgfrac):
    g3d, cam = scene(n, W, H, float(W), bgfrac=bgfrac)
    g2d = O.project_all(g3d, cam)
    bg = (0.1, 0.2, 0.3)
    ref = _oracle_render(variant, g2d, W, H, pw, ph, bg)
    got, _ = _gpu_render(variant, g2d, W, H, pw, ph, bg, N.ALPHA_EXACT)
    assert np.array_equal(got["contrib"], ref["contrib"])
    assert np.array_equal(got["term"], ref["term"])
    assert np.array_equal(got["final_t"].view(np.uint32), ref["final_t"].view(np.uint32))
    assert np.array_equal(got["alpha"].view(np.uint32), ref["alpha"].view(np.uint32))
    if variant in (0, 1, 4):  # pixel-wise: bit-exact colour/depth too
        assert np.array_equal(got["color"].view(np.uint32), ref["color"].view(np.uint32))
        assert np.array_equal(got["depth"].view(np.uint32), ref["depth"].view(np.uint32))
    else:
        assert np.max(np.abs(got["color"] - ref["color"])) <= 1e-6
        assert np.max(np.abs(got["depth"] - ref["depth"]) / np.maximum(1, np.abs(ref["depth"]))) <= 1e-6
    if variant == 3:
        # the B200 FineGrainedCombined blends with serial weights: it equals
        # render_reference (not only render_gaussianwise) to double-sum order
        ref0 = _oracle_render(0, g2d, W, H, pw, ph, bg)
        assert np.array_equal(got["contrib"], ref0["contrib"]) and np.array_equal(got["term"], ref0["term"])
        assert np.max(np.abs(got["color"] - ref0["color"])) <= 1e-6
        same = np.mean(got["color"].view(np.uint32) == ref0["color"].view(np.uint32))
        assert same > 0.99, same


@pytest.mark.parametrize("variant", range(5))
def test_render_fast_tolerance(variant):
    W, H, pw, ph = 256, 256, 16, 16
    g3d, cam = scene(20000, W, H, 256.0, bgfrac=0.12)
    g2d = O.project_all(g3d, cam)
    bg = (0.1, 0.2, 0.3)
    ref = _oracle_render(variant, g2d, W, H, pw, ph, bg)
    got, _ = _gpu_render(variant, g2d, W, H, pw, ph, bg, N.ALPHA_FAST)
    match = (got["contrib"] == ref["contrib"]) & (got["term"] == ref["term"])
    frac_mismatch = 1.0 - match.mean()
    assert frac_mismatch < 2e-3, frac_mismatch
    col_err = np.abs(got["color"] - ref["color"]).reshape(-1, 3).max(axis=1)
    assert col_err[match].max() <= 1e-4
    assert np.abs(got["final_t"] - ref["final_t"])[match].max() <= 1e-4


def test_render_empty_scene_is_background():
    W, H = 64, 48
    g2d = np.zeros(0, dtype=O.G2D_DTYPE)
    for v in range(5):
        got, _ = _gpu_render(v, g2d, W, H, 16, 16, (0.25, 0.5, 0.75), N.ALPHA_EXACT)
        assert np.allclose(got["color"].reshape(-1, 3), [0.25, 0.5, 0.75])
        assert (got["final_t"] == 1).all() and (got["contrib"] == 0).all() and (got["term"] == 0).all()


def test_frame_work_counts():
    W, H, pw, ph = 256, 256, 16, 16
    g3d, cam = scene(10000, W, H, 256.0, bgfrac=0.5)
    g2d = O.project_all(g3d, cam)
    got, b = _gpu_render(0, g2d, W, H, pw, ph, (0, 0, 0), N.ALPHA_EXACT)
    f = api.DeviceFrame.empty(W, H, DEV)
    f.term.copy_(torch.from_numpy(got["term"]))
    f.contrib.copy_(torch.from_numpy(got["contrib"]))
    e, c = api.frame_work(f, b, pw, ph)
    rg = b.tile_ranges.cpu().numpy().view(np.uint32)
    lens = (rg[1::2] - rg[0::2]).astype(np.int64)
    py, px = np.divmod(np.arange(W * H), W)
    tile = (py // ph) * (W // pw) + px // pw
    cons = np.where(got["term"] > 0, got["term"], lens[tile])
    assert e == int(cons.sum()) and c == int(got["contrib"].sum())


def test_pipeline_end_to_end_matches_oracle():
    W, H, pw, ph = 320, 192, 16, 16
    g3d, cam = scene(15000, W, H, 320.0)
    ref_g2d = O.project_all(g3d, cam)
    ref = _oracle_render(3, ref_g2d, W, H, pw, ph, (0, 0, 0))
    pipe = api.Pipeline(W, H, pw, ph, DEV, N.ALPHA_EXACT)
    frame, v = pipe.forward(api.g3d_to_device(g3d), len(g3d), ncam(cam), variant="FineGrainedCombined")
    got = frame.to_numpy()
    assert np.array_equal(got["contrib"], ref["contrib"]) and np.array_equal(got["term"], ref["term"])
    assert np.max(np.abs(got["color"] - ref["color"])) <= 1e-6


def test_golden_digests_on_gpu():
    """The whole GPU pipeline reproduces the frozen oracle fixture digests."""
    import json
    import os

    from golden.gen_golden import FIXTURES

    with open(os.path.join(os.path.dirname(__file__), "golden", "digests.json")) as fh:
        frozen = json.load(fh)
    for name, (n, W, H, f, bgf, pw, ph, bg) in FIXTURES.items():
        cam = O.make_camera(focal=(f, f), width=W, height=H)
        g3d = O.gen_clustered_scene(n, cam, bgfrac=bgf)
        fz = frozen[name]
        s = api.project_all(api.g3d_to_device(g3d), n, ncam(cam))
        assert O.fnv1a64(api.splats_to_g2d(s)) == fz["g2d"], name
        b = api.bin_tiles(s, W, H, pw, ph)
        assert O.fnv1a64(b.point_list.cpu().numpy().view(np.uint32)) == fz["point_list"], name
        assert O.fnv1a64(b.tile_ranges.cpu().numpy().view(np.uint32)) == fz["tile_ranges"], name
        st = api.tile_load_histogram(b)
        for v in (0, 1, 4):  # pixel-wise variants: every plane bit-exact
            f_ = api.render_forward(v, s, b, W, H, pw, ph, bg, N.ALPHA_EXACT, st.task_order).to_numpy()
            for k, dg in fz["render_reference"].items():
                assert O.fnv1a64(f_[k]) == dg, (name, v, k)
        f2 = api.render_forward(2, s, b, W, H, pw, ph, bg, N.ALPHA_EXACT, st.task_order).to_numpy()
        for k in ("alpha", "final_t", "contrib", "term"):
            assert O.fnv1a64(f2[k]) == fz["render_gaussianwise"][k], (name, k)


@pytest.mark.parametrize("after,remain", [("0", "1"), ("32", "64"), ("100000000", "100000000")])
def test_fine_donation_path(after, remain, monkeypatch):
    """FineGrainedCombined's tail hand-off (live pixels parked mid-list and
    finished Gaussian-wise by k_render_donated), forced on with tiny
    thresholds, keeps the exact semantics; the last case disables it."""
    monkeypatch.setenv("BS_FINE_DONATE_AFTER", after)
    monkeypatch.setenv("BS_FINE_DONATE_MIN", remain)
    W, H, pw, ph = 192, 128, 16, 16
    g3d, cam = scene(8000, W, H, 192.0, bgfrac=0.12)
    g2d = O.project_all(g3d, cam)
    bg = (0.1, 0.2, 0.3)
    ref = _oracle_render(0, g2d, W, H, pw, ph, bg)
    for mode in (N.ALPHA_EXACT, N.ALPHA_FAST):
        got, _ = _gpu_render(3, g2d, W, H, pw, ph, bg, mode)
        if mode == N.ALPHA_EXACT:
            assert np.array_equal(got["contrib"], ref["contrib"]) and np.array_equal(got["term"], ref["term"])
            assert np.array_equal(got["final_t"].view(np.uint32), ref["final_t"].view(np.uint32))
            assert np.max(np.abs(got["color"] - ref["color"])) <= 1e-6
        else:
            match = (got["contrib"] == ref["contrib"]) & (got["term"] == ref["term"])
            assert 1.0 - match.mean() < 2e-3
            err = np.abs(got["color"] - ref["color"]).reshape(-1, 3).max(axis=1)
            assert err[match].max() <= 1e-4


@pytest.mark.parametrize("n,bgfrac", [(60, 1.0), (8000, 0.12)])
def test_frame_pipeline_device_selection(n, bgfrac):
    """bs_render_frame_device with variant=-1: the variant is chosen on the
    device (bs_select_variant_device) and only that kernel renders; the frame
    equals the oracle's render of the chosen variant and the choice equals the
    host selector's on the same tile statistics."""
    W = H = 256
    g3d, cam = scene(n, W, H, 256.0, bgfrac=bgfrac)
    g2d = O.project_all(g3d, cam)
    pl, rg = O.bin_tiles(g2d, W, H, 16, 16)
    fp = api.FramePipeline(W, H, 16, 16, DEV, N.ALPHA_EXACT)
    frame, fi = fp.forward(api.g3d_to_device(g3d), n, ncam(cam), variant="auto", bg=(0.1, 0.2, 0.3), info=True)
    got = frame.to_numpy()
    v_host = N.lib().bs_select_variant(C.byref(fi.stats), W, H, 16, 16, api.sm_count())
    assert fi.variant == v_host and fi.k == len(pl)
    ref = O.render(fi.variant, pl, rg, g2d, W, H, 16, 16, (0.1, 0.2, 0.3), lazy=True, threads=0)
    for k in ("contrib", "term", "final_t", "alpha"):
        assert np.array_equal(got[k], ref[k]), k
    assert float(np.abs(got["color"] - ref["color"]).max()) <= 1e-6
    # forced variants through the same context
    for v in (BS_FG, BS_SMO):
        frame, fi2 = fp.forward(api.g3d_to_device(g3d), n, ncam(cam), variant=v, bg=(0.1, 0.2, 0.3), info=True)
        assert fi2.variant == v
        assert np.array_equal(frame.to_numpy()["contrib"], ref["contrib"])
    fp.close()


BS_FG, BS_SMO = 3, 4


def _len_bucket(c):
    out = np.empty(len(c), dtype=np.int64)
    for i, x in enumerate(c.tolist()):
        v = x + 1
        e = v.bit_length() - 1
        out[i] = v if e < 3 else min(8 * e + ((v >> (e - 3)) & 7), 255)
    return out


@pytest.mark.parametrize("W,H,n", [(1920, 1080, 100_000), (3840, 2160, 20_000), (64, 64, 0)])
def test_tile_order_lpt_buckets(W, H, n):
    """bs_tile_order: sum/max/mean/nonempty as tile_load_histogram, and the
    task order = stable sort by eighth-octave length bucket, descending."""
    cols, rows = (W + 15) // 16, (H + 15) // 16
    T = cols * rows
    if n:
        g3d, cam = scene(n, W, H, W / 2.0)
        g2d = O.project_all(g3d, cam)
    else:
        g2d = np.zeros(0, dtype=O.G2D_DTYPE)
    pl, rg = O.bin_tiles(g2d, W, H, 16, 16)
    ref = O.tile_load_histogram(rg, cols, rows)
    rgd = torch.from_numpy(rg.view(np.int32).copy()).to(DEV)
    hist = torch.zeros(64, dtype=torch.uint8, device=DEV)
    order = torch.empty(T, dtype=torch.int32, device=DEV)
    N.call("bs_tile_order", rgd.data_ptr(), T, hist.data_ptr(), order.data_ptr(), api._stream(DEV))
    h = N.TileHistogram.from_buffer_copy(hist.cpu().numpy().tobytes()[: C.sizeof(N.TileHistogram)])
    assert h.total == len(pl) and h.max == ref["max"] and h.mean == ref["mean"] and h.tiles == T
    assert h.nonempty == int((ref["counts"] > 0).sum())
    b = _len_bucket(ref["counts"])
    exp = np.lexsort((np.arange(T), -b))
    assert np.array_equal(order.cpu().numpy(), exp)


def test_frame_pipeline_async_overflow_rerun():
    """Async mode: the first frame's K exceeds the initial point_list
    capacity (64 per Gaussian), so it is rendered again at the next sync point
    with a grown capacity; the final output equals the oracle's, and later
    frames need no re-render."""
    W = H = 512
    n = 300
    g3d, cam = scene(n, W, H, 4096.0, bgfrac=1.0)
    g2d = O.project_all(g3d, cam)
    pl, rg = O.bin_tiles(g2d, W, H, 16, 16)
    # the initial capacity overflows, with 16x16 lists and with the frame
    # pipeline's 32x32 super-tile lists alike
    assert len(pl) > 64 * n and len(O.bin_tiles(g2d, W, H, 32, 32)[0]) > 64 * n
    fp = api.FramePipeline(W, H, 16, 16, DEV, N.ALPHA_EXACT, async_mode=True)
    d = api.g3d_to_device(g3d)
    fp.forward(d, n, ncam(cam), variant=BS_FG, bg=(0.1, 0.2, 0.3))
    assert fp.sync() == 1
    ref = O.render(BS_FG, pl, rg, g2d, W, H, 16, 16, (0.1, 0.2, 0.3), lazy=True, threads=0)
    got = fp.frame.to_numpy()
    for k in ("contrib", "term", "final_t"):
        assert np.array_equal(got[k], ref[k]), k
    for _ in range(3):
        fp.forward(d, n, ncam(cam), variant="auto", bg=(0.1, 0.2, 0.3))
    assert fp.sync() == 1
    got = fp.frame.to_numpy()
    assert np.array_equal(got["contrib"], ref["contrib"]) and np.array_equal(got["final_t"], ref["final_t"])
    fp.close()


def test_frame_pipeline_super_overflow_rerun():
    """The async overflow path on a super-tile frame (1024x1024): the first
    frame's super-tile K exceeds the initial capacity, the frame is rendered
    again at the sync point, and equals the oracle's 16x16 render."""
    W = H = 1024
    n = 300
    g3d, cam = scene(n, W, H, 4096.0, bgfrac=1.0)
    g2d = O.project_all(g3d, cam)
    pl, rg = O.bin_tiles(g2d, W, H, 16, 16)
    assert len(O.bin_tiles(g2d, W, H, 32, 32)[0]) > 64 * n
    fp = api.FramePipeline(W, H, 16, 16, DEV, N.ALPHA_EXACT, async_mode=True)
    fp.forward(api.g3d_to_device(g3d), n, ncam(cam), variant=BS_FG, bg=(0.1, 0.2, 0.3))
    assert fp.sync() == 1
    mode = C.c_int32(0)
    N.call("bs_context_list_mode", fp.ctx, C.byref(mode))
    assert mode.value == 1
    ref = O.render(BS_FG, pl, rg, g2d, W, H, 16, 16, (0.1, 0.2, 0.3), lazy=True, threads=0)
    got = fp.frame.to_numpy()
    for k in ("contrib", "term", "final_t"):
        assert np.array_equal(got[k], ref[k]), k
    fp.close()


def test_frame_pipeline_async_two_in_flight_capacity_growth():
    """Two async frames in flight: checking the first one grows the capacity
    (first-frame calibration to 3x its K), and the second one had overflowed
    the capacity it was SORTED with.  Its K must be checked against that
    capacity, not the grown one, so it is rendered again."""
    W = H = 512
    n = 300
    g3d = O.gen_clustered_scene(n, O.make_camera(focal=(1500, 1500), width=W, height=H), bgfrac=1.0)
    cams = [O.make_camera(focal=(f, f), width=W, height=H) for f in (1000.0, 1500.0)]
    refs, ks = [], []
    for cam in cams:
        g2d = O.project_all(g3d, cam)
        pl, rg = O.bin_tiles(g2d, W, H, 16, 16)
        ks.append(len(pl))
        refs.append(O.render(BS_FG, pl, rg, g2d, W, H, 16, 16, (0.1, 0.2, 0.3), lazy=True, threads=0))
    # frame 0 fits the initial capacity (64 per Gaussian), frame 1 does not,
    # but it fits the capacity frame 0's check grows to (3 K0)
    assert ks[0] < 64 * n < ks[1] <= 3 * ks[0]
    fp = api.FramePipeline(W, H, 16, 16, DEV, N.ALPHA_EXACT, async_mode=True)
    d = api.g3d_to_device(g3d)
    frames = [api.DeviceFrame.empty(W, H, DEV) for _ in range(3)]
    for i, cam in enumerate([cams[0], cams[1], cams[0]]):
        fp.frame = frames[i]
        fp.forward(d, n, ncam(cam), variant=BS_FG, bg=(0.1, 0.2, 0.3))
    assert fp.sync() >= 1
    for i, ref in ((0, refs[0]), (1, refs[1]), (2, refs[0])):
        got = frames[i].to_numpy()
        for k in ("contrib", "term", "final_t"):
            assert np.array_equal(got[k], ref[k]), (i, k)
    fp.close()


def test_frame_pipeline_sync_frame_keeps_pending_k():
    """A synchronous frame (a grid the async path does not take) while an
    async frame is pending uses its own K slot: the pending frame's K check
    still reads its own count."""
    W = H = 512
    n = 300
    g3d = O.gen_clustered_scene(n, O.make_camera(focal=(1500, 1500), width=W, height=H), bgfrac=1.0)
    cam = O.make_camera(focal=(1500.0, 1500.0), width=W, height=H)
    g2d = O.project_all(g3d, cam)
    pl, rg = O.bin_tiles(g2d, W, H, 16, 16)
    assert len(pl) > 64 * n  # the async frame overflows the initial capacity
    ref = O.render(BS_FG, pl, rg, g2d, W, H, 16, 16, (0.1, 0.2, 0.3), lazy=True, threads=0)
    fp = api.FramePipeline(W, H, 16, 16, DEV, N.ALPHA_EXACT, async_mode=True)
    d = api.g3d_to_device(g3d)
    fa = api.DeviceFrame.empty(W, H, DEV)
    fp.frame = fa
    fp.forward(d, n, ncam(cam), variant=BS_FG, bg=(0.1, 0.2, 0.3))
    # a frame in between through the same context on a 131,072-tile grid
    # (beyond the chunked scatter: the synchronous body), few instances
    big = O.make_camera(focal=(10.0, 10.0), width=8192, height=4096)
    assert not N.lib().bs_bin_async_supported(8192, 4096, 16, 16)
    fp.frame = api.DeviceFrame.empty(8192, 4096, DEV)
    fp.forward(d, n, ncam(big), variant=BS_FG, bg=(0.1, 0.2, 0.3), info=True)
    fp.sync()
    got = fa.to_numpy()
    for k in ("contrib", "term", "final_t"):
        assert np.array_equal(got[k], ref[k]), k
    fp.close()


def test_frame_pipeline_runs_on_torch_stream():
    """FramePipeline enqueues on torch's current stream: reading the frame on
    that stream right after forward (no explicit sync) sees the finished frame."""
    W, H = 960, 540
    g3d, cam = scene(100_000, W, H, 500.0)
    d = api.g3d_to_device(g3d)
    fp = api.FramePipeline(W, H, 16, 16, DEV, N.ALPHA_EXACT, async_mode=True)
    fp.forward(d, len(g3d), ncam(cam), variant=BS_FG)
    fp.sync()
    ref = fp.frame.color.clone()
    for _ in range(3):
        fp.frame.color.zero_()
        fp.forward(d, len(g3d), ncam(cam), variant=BS_FG)
        got = fp.frame.color.cpu()  # stream-ordered read on torch's current stream
        assert torch.equal(got, ref.cpu())
    fp.close()


def _rect_rule(g2d, W, H, pw, ph):
    """The reference's tile rectangle (src/preprocess.cpp:81-92) in float32,
    vectorised: (tx0, tx1, ty0, ty1, touches)."""
    x, y = g2d["x"], g2d["y"]
    rr = np.ceil(g2d["radius"]).astype(np.float32)
    x0, x1, y0, y1 = x - rr, x + rr, y - rr, y + rr
    cols, rows = (W + pw - 1) // pw, (H + ph - 1) // ph
    ok = ~((x1 < 0) | (y1 < 0) | (x0 >= np.float32(W)) | (y0 >= np.float32(H)))
    with np.errstate(invalid="ignore", over="ignore"):
        tx0 = np.maximum(0, np.floor(x0 / np.float32(pw))).astype(np.int64)
        tx1 = np.minimum(cols - 1, np.floor(x1 / np.float32(pw))).astype(np.int64)
        ty0 = np.maximum(0, np.floor(y0 / np.float32(ph))).astype(np.int64)
        ty1 = np.minimum(rows - 1, np.floor(y1 / np.float32(ph))).astype(np.int64)
    return tx0, tx1, ty0, ty1, ok & (tx0 <= tx1) & (ty0 <= ty1)


@pytest.mark.parametrize("mode", [N.ALPHA_EXACT])
def test_c4_tile_sampled(mode):
    """C4 at full size (3840x2160, 3M clustered Gaussians, K ~ 5e8):
    tile-sampled parity (the 64 longest tiles + 1 % random tiles,
    seed 42).  For every sampled tile the GPU list must be exactly the splats
    whose rectangle contains it, in (depth, index) order, and the
    FineGrainedCombined frame must equal the oracle's render of those lists."""
    W, H, f, n = 3840, 2160, 2000.0, 3_000_000
    cam = N.make_camera(None, (f, f), W, H)
    g3d = api.gen_clustered_scene(n, cam)
    fp = api.FramePipeline(W, H, 16, 16, DEV, mode)
    frame, fi = fp.forward(api.g3d_to_device(g3d), n, cam, variant=BS_FG, bg=(0.1, 0.2, 0.3), info=True)
    got = frame.to_numpy()
    ocam = O.Camera.from_buffer_copy(bytes(cam))
    g2d = O.project_all(g3d.view(O.G3D_DTYPE), ocam)
    assert fi.n_visible == len(g2d)
    cols, rows = 240, 135
    T = cols * rows
    # the pipeline's binning (same context buffers) for the sampled tiles
    pipe = api.Pipeline(W, H, 16, 16, DEV, mode)
    pipe.forward(api.g3d_to_device(g3d), n, cam, variant=BS_FG)
    b = pipe.last_binning
    assert b.k == fi.k
    rg = b.tile_ranges.cpu().numpy().view(np.uint32)
    lens = (rg[1::2] - rg[0::2]).astype(np.int64)
    rng = np.random.default_rng(42)
    tiles = np.unique(np.concatenate([np.argsort(-lens, kind="stable")[:64], rng.choice(T, T // 100, replace=False)]))
    tx0, tx1, ty0, ty1, ok = _rect_rule(g2d, W, H, 16, 16)
    key = np.lexsort((np.arange(len(g2d)), g2d["depth"]))  # (depth, index) order
    rank = np.empty(len(g2d), np.int64)
    rank[key] = np.arange(len(g2d))
    pl_dev = b.point_list
    sub_pl, sub_rg = [], np.zeros(2 * T, np.uint32)
    pos = 0
    for t in tiles.tolist():
        tx, ty = t % cols, t // cols
        lst = pl_dev[int(rg[2 * t]):int(rg[2 * t + 1])].cpu().numpy().view(np.uint32)
        inside = np.nonzero(ok & (tx0 <= tx) & (tx <= tx1) & (ty0 <= ty) & (ty <= ty1))[0]
        exp = inside[np.argsort(rank[inside], kind="stable")]
        assert np.array_equal(lst, exp.astype(np.uint32)), t
        sub_rg[2 * t], sub_rg[2 * t + 1] = pos, pos + len(lst)
        sub_pl.append(lst)
        pos += len(lst)
    ref = O.render(BS_FG, np.concatenate(sub_pl), sub_rg, g2d, W, H, 16, 16, (0.1, 0.2, 0.3), lazy=True, threads=0,
                   tiles=tiles.astype(np.int32))
    px = np.zeros((H, W), bool)
    for t in tiles.tolist():
        px[(t // cols) * 16:(t // cols) * 16 + 16, (t % cols) * 16:(t % cols) * 16 + 16] = True
    m = px.reshape(-1)
    for k in ("contrib", "term", "final_t", "alpha"):
        assert np.array_equal(got[k][m], ref[k][m]), k
    assert float(np.abs(got["color"].reshape(-1, 3)[m] - ref["color"].reshape(-1, 3)[m]).max()) <= 1e-6
    fp.close()


def test_frame_pipeline_graph_replay_matches():
    """CUDA-graph mode: frames replayed from the captured graph (new camera
    each time) equal the same frames rendered launch by launch."""
    W, H, f, n = 960, 540, 500.0, 200_000
    cams = [N.make_camera(sharding.orbit_view(k * 9), (f, f), W, H) for k in range(7)]
    g3d = api.gen_clustered_scene(n, cams[0])
    d = api.g3d_to_device(g3d)
    ref = []
    fp = api.FramePipeline(W, H, 16, 16, DEV, N.ALPHA_EXACT, async_mode=True)
    for cam in cams:
        fp.forward(d, n, cam)
        fp.sync()
        ref.append(fp.frame.to_numpy())
    fp.close()
    fg = api.FramePipeline(W, H, 16, 16, DEV, N.ALPHA_EXACT, async_mode=True, graphs=True)
    for i, cam in enumerate(cams):
        fg.forward(d, n, cam)
        fg.sync()
        got = fg.frame.to_numpy()
        for k in ("color", "contrib", "term", "final_t", "depth"):
            assert np.array_equal(got[k], ref[i][k]), (i, k)
    assert fg.graph_launches() >= len(cams) - 2  # the first frame (and captures) run plainly
    fg.close()


class _DevArray:
    """A raw device pointer viewed through __cuda_array_interface__."""

    def __init__(self, ptr, count, typestr):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3}


def test_render_views_batch_matches():
    """bs_render_views: views enqueued round-robin over two contexts by one
    native call (with per-view L2 flushes) equal the same views rendered one
    call at a time; checked on each context's last view, over several batches
    so graph capture and replay both run."""
    W, H, f, n = 960, 540, 500.0, 200_000
    cams = [N.make_camera(sharding.orbit_view(k * 11), (f, f), W, H) for k in range(8)]
    g3d = api.gen_clustered_scene(n, cams[0])
    d = api.g3d_to_device(g3d)
    ref = []
    fp = api.FramePipeline(W, H, 16, 16, DEV, N.ALPHA_EXACT)
    for cam in cams:
        fp.forward(d, n, cam)
        fp.sync()
        ref.append(fp.frame.to_numpy())
    fp.close()
    streams = [torch.cuda.Stream(device=DEV) for _ in range(2)]
    fps = []
    for s_ in streams:
        with torch.cuda.stream(s_):
            fps.append(api.FramePipeline(W, H, 16, 16, DEV, N.ALPHA_EXACT, async_mode=True, graphs=True))
    ctxs = (C.c_void_p * 2)(*[q.ctx.value for q in fps])
    flush = [torch.empty(1 << 20, dtype=torch.uint8, device=DEV) for _ in range(2)]
    flush_arr = (C.c_void_p * 2)(*[t.data_ptr() for t in flush])
    cam_arr = (N.Camera * len(cams))(*cams)
    bg = (C.c_float * 3)(0.0, 0.0, 0.0)
    P = W * H
    for batch in ([0, 1, 2, 3], [4, 5, 6, 7], [7, 2, 5, 0], [3, 6]):
        ids = (C.c_int32 * len(batch))(*batch)
        N.call("bs_render_views", ctxs, 2, C.c_void_p(d.data_ptr()), n, cam_arr, ids, len(batch), 16, 16, -1, bg,
               flush_arr, 1 << 20)
        for q in fps:
            q.sync()
        torch.cuda.synchronize()
        for ci in range(2):
            last = batch[max(j for j in range(len(batch)) if j % 2 == ci)]
            fo = N.FrameOut()
            N.call("bs_context_frame", ctxs[ci], C.byref(fo))
            color = torch.as_tensor(_DevArray(fo.color, 3 * P, "<f4"), device=DEV).cpu().numpy()
            contrib = torch.as_tensor(_DevArray(fo.contrib, P, "<i4"), device=DEV).cpu().numpy()
            final_t = torch.as_tensor(_DevArray(fo.final_t, P, "<f4"), device=DEV).cpu().numpy()
            assert np.array_equal(color, ref[last]["color"].reshape(-1)), (batch, ci)
            assert np.array_equal(contrib, ref[last]["contrib"].reshape(-1)), (batch, ci)
            assert np.array_equal(final_t, ref[last]["final_t"].reshape(-1)), (batch, ci)
    assert sum(q.graph_launches() for q in fps) > 0
    for q in fps:
        q.close()


def test_frame_pipeline_super_lists_match_tile_lists():
    """Frames >= 1 Mpixel take the super-tile path (lists at 32x32, members
    kept per 16x16 tile); with graphs and async frames they equal the
    stage-by-stage pipeline on 16x16 lists."""
    W, H, f, n = 1280, 832, 700.0, 150_000
    cams = [N.make_camera(sharding.orbit_view(k * 13), (f, f), W, H) for k in range(5)]
    g3d = api.gen_clustered_scene(n, cams[0])
    d = api.g3d_to_device(g3d)
    pipe = api.Pipeline(W, H, 16, 16, DEV, N.ALPHA_EXACT)
    ref = []
    for cam in cams:
        fr, _ = pipe.forward(d, n, cam, variant=BS_FG)
        torch.cuda.synchronize()
        ref.append(fr.to_numpy())
    fp = api.FramePipeline(W, H, 16, 16, DEV, N.ALPHA_EXACT, async_mode=True, graphs=True)
    for i, cam in enumerate(cams):
        fp.forward(d, n, cam, variant=BS_FG)
        fp.sync()
        got = fp.frame.to_numpy()
        for k in ("contrib", "term"):
            assert np.array_equal(got[k], ref[i][k]), (i, k)
        for k in ("final_t", "alpha"):
            assert np.array_equal(got[k].view(np.uint32), ref[i][k].view(np.uint32)), (i, k)
        assert np.max(np.abs(got["color"] - ref[i]["color"])) <= 1e-6
        assert np.max(np.abs(got["depth"] - ref[i]["depth"]) / np.maximum(1, np.abs(ref[i]["depth"]))) <= 1e-6
    _, fi = fp.forward(d, n, cams[0], variant=BS_FG, info=True)
    pipe.forward(d, n, cams[0], variant=BS_FG)
    assert fi.k == pipe.last_binning.k  # info reports the 16x16 instance count
    fp.close()


def test_frame_pipeline_super_lists_fast_mode():
    """BS_ALPHA_FAST through the super-tile frame path: RGB / T within 1e-4 of
    the oracle on pixels whose contrib / term match, mismatches rare."""
    W, H, f, n = 1280, 832, 700.0, 60_000
    cam = N.make_camera(None, (f, f), W, H)
    g3d = api.gen_clustered_scene(n, cam)
    g2d = O.project_all(g3d.view(O.G3D_DTYPE), O.Camera.from_buffer_copy(bytes(cam)))
    pl, rg = O.bin_tiles(g2d, W, H, 16, 16)
    bg = (0.1, 0.2, 0.3)
    ref = O.render(BS_FG, pl, rg, g2d, W, H, 16, 16, bg, lazy=True, threads=0)
    fp = api.FramePipeline(W, H, 16, 16, DEV, N.ALPHA_FAST, async_mode=True)
    fp.forward(api.g3d_to_device(g3d), n, cam, variant=BS_FG, bg=bg)
    fp.sync()
    mode = C.c_int32(0)
    N.call("bs_context_list_mode", fp.ctx, C.byref(mode))
    assert mode.value == 1
    got = fp.frame.to_numpy()
    match = (got["contrib"] == ref["contrib"]) & (got["term"] == ref["term"])
    assert 1.0 - match.mean() < 2e-3
    err = np.abs(got["color"] - ref["color"]).reshape(-1, 3).max(axis=1)
    assert err[match].max() <= 1e-4
    assert np.abs(got["final_t"] - ref["final_t"])[match].max() <= 1e-4
    fp.close()


def test_host_async_pipeline_matches():
    """bs_render_frame_host_async: frames uploaded / rendered / downloaded on
    three streams equal the synchronous host-buffer frames."""
    W, H, f, n = 480, 270, 250.0, 40_000
    cams = [N.make_camera(sharding.orbit_view(k * 7), (f, f), W, H) for k in range(6)]
    g3d = api.gen_clustered_scene(n, cams[0])
    host = torch.from_numpy(np.ascontiguousarray(g3d).view(np.uint8).reshape(-1).copy()).pin_memory()
    P = W * H
    bg = (C.c_float * 3)(0.1, 0.2, 0.3)

    def planes():
        return ([torch.empty(3 * P, dtype=torch.float32).pin_memory()] +
                [torch.empty(P, dtype=torch.float32).pin_memory() for _ in range(3)] +
                [torch.empty(P, dtype=torch.int32).pin_memory() for _ in range(2)])

    ref = []
    ctx = C.c_void_p()
    N.call("bs_context_create", C.byref(ctx), N.ALPHA_EXACT)
    for cam in cams:
        out = planes()
        N.call("bs_render_frame_host", ctx, host.data_ptr(), n, C.byref(cam), 16, 16, -1, bg,
               *[o.data_ptr() for o in out], None)
        ref.append([o.clone() for o in out])
    N.call("bs_context_destroy", ctx)
    ctx = C.c_void_p()
    N.call("bs_context_create", C.byref(ctx), N.ALPHA_EXACT)
    N.call("bs_context_set_async", ctx, 1)
    outs = [planes() for _ in cams]
    for cam, out in zip(cams, outs):
        N.call("bs_render_frame_host_async", ctx, host.data_ptr(), n, C.byref(cam), 16, 16, -1, bg,
               *[o.data_ptr() for o in out])
    N.call("bs_context_sync", ctx, None)
    N.call("bs_context_destroy", ctx)
    for i, (a, r) in enumerate(zip(outs, ref)):
        for k in range(6):
            assert torch.equal(a[k], r[k]), (i, k)


def test_two_pipelines_on_two_streams():
    """Two Pipelines rendering FineGrainedCombined concurrently on two torch
    streams: each owns its render workspace (work-queue counters, tail
    hand-off slots), so neither frame is corrupted."""
    W, H = 480, 320
    scenes = []
    for seed, bgf in ((1, 0.12), (2, 0.6)):
        g3d, cam = scene(40000, W, H, 480.0, bgfrac=bgf, seed=seed)
        g2d = O.project_all(g3d, cam)
        scenes.append((g3d, cam, _oracle_render(3, g2d, W, H, 16, 16, (0.1, 0.2, 0.3))))
    pipes = [api.Pipeline(W, H, 16, 16, DEV, N.ALPHA_EXACT) for _ in scenes]
    streams = [torch.cuda.Stream() for _ in scenes]
    devs = [api.g3d_to_device(g) for g, _, _ in scenes]
    for _ in range(4):
        for p, st, d, (g3d, cam, _) in zip(pipes, streams, devs, scenes):
            with torch.cuda.stream(st):
                p.forward(d, len(g3d), ncam(cam), variant="FineGrainedCombined", bg=(0.1, 0.2, 0.3))
        torch.cuda.synchronize()
        for p, (_, _, ref) in zip(pipes, scenes):
            got = p.frame.to_numpy()
            assert np.array_equal(got["contrib"], ref["contrib"]) and np.array_equal(got["term"], ref["term"])
            assert np.array_equal(got["final_t"], ref["final_t"])


def test_render_views_host_batch_matches():
    """bs_render_views_host: one scene upload per call, views round-robin over
    two async contexts, every view's planes downloaded to its own host
    buffers; three calls back to back (the alternating scene buffers), each
    view equal to the oracle's render of that view."""
    W, H, f, n = 640, 480, 600.0, 30000
    g3d, cam0 = scene(n, W, H, f)
    views = [3, 17, 40, 63, 9]
    cams = [N.make_camera(sharding.orbit_view(k), (f, f), W, H) for k in range(64)]
    refs = {}
    for k in views:
        oc = O.Camera.from_buffer_copy(bytes(cams[k]))
        g2d = O.project_all(g3d, oc)
        pl, rg = O.bin_tiles(g2d, W, H, 16, 16)
        refs[k] = O.render(0, pl, rg, g2d, W, H, 16, 16, (0.1, 0.2, 0.3), lazy=True, threads=0)
    ctxs = []
    for _ in range(2):
        cx = C.c_void_p()
        N.call("bs_context_create", C.byref(cx), N.ALPHA_EXACT)
        N.call("bs_context_set_async", cx, 1)
        ctxs.append(cx)
    P = W * H
    host = np.ascontiguousarray(g3d)
    ctx_arr = (C.c_void_p * 2)(*[c.value for c in ctxs])
    cam_arr = (N.Camera * 64)(*cams)
    ids = (C.c_int32 * len(views))(*views)
    bgc = (C.c_float * 3)(0.1, 0.2, 0.3)
    calls = []
    for _ in range(3):
        outs = [[np.zeros(3 * P, np.float32)] + [np.zeros(P, np.float32) for _ in range(3)] +
                [np.zeros(P, np.int32) for _ in range(2)] for _ in views]
        ptrs = (C.c_void_p * (6 * len(views)))(*[o.ctypes.data for v in outs for o in v])
        N.call("bs_render_views_host", ctx_arr, 2, host.ctypes.data, n, cam_arr, ids, len(views), 16, 16, -1, bgc,
               ptrs)
        calls.append((outs, ptrs))
    for c in ctxs:
        N.call("bs_context_sync", c, None)
        N.call("bs_context_destroy", c)
    for outs, _ in calls:
        for k, o in zip(views, outs):
            ref = refs[k]
            assert np.array_equal(o[4], ref["contrib"]) and np.array_equal(o[5], ref["term"]), k
            assert np.array_equal(o[3], ref["final_t"]) and np.array_equal(o[1], ref["alpha"]), k
            assert float(np.abs(o[0] - ref["color"]).max()) <= 1e-6, k


def test_gaussianwise_windowed_bit_exact_colour():
    """BS_GW_WINDOWED=1 selects the GaussianWise kernel that keeps the
    reference's fixed 32-entry windows (no sub-tile cull): every plane,
    colour and depth included, equals render_gaussianwise bit for bit.  (The
    knob is read once per process, hence the subprocess.)"""
    import os
    import subprocess
    import sys
    code = r"""
import sys, numpy as np
sys.path.insert(0, "tests")
import oracle_lib as O
from paper_2412_17378_b200 import _native as N, api
for (W, H, pw, ph, n, bgf) in [(256, 256, 16, 16, 10000, 1.0), (192, 128, 16, 8, 6000, 0.12), (90, 70, 8, 8, 2000, 0.3)]:
    cam = O.make_camera(focal=(float(W), float(W)), width=W, height=H)
    g2d = O.project_all(O.gen_clustered_scene(n, cam, bgfrac=bgf), cam)
    pl, rg = O.bin_tiles(g2d, W, H, pw, ph)
    ref = O.render(2, pl, rg, g2d, W, H, pw, ph, (0.1, 0.2, 0.3), lazy=True, threads=0)
    s = api.splats_from_g2d(g2d, "cuda")
    b = api.bin_tiles(s, W, H, pw, ph)
    st = api.tile_load_histogram(b)
    got = api.render_forward(2, s, b, W, H, pw, ph, (0.1, 0.2, 0.3), N.ALPHA_EXACT, st.task_order).to_numpy()
    for k in ("color", "alpha", "depth", "final_t", "contrib", "term"):
        assert got[k].tobytes() == ref[k].tobytes(), (W, H, k)
print("windowed ok")
"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=dict(os.environ, BS_GW_WINDOWED="1"),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "windowed ok" in r.stdout, r.stdout + r.stderr[-2000:]
