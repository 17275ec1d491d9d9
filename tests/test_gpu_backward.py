"""SURVEY 8f(4) backward render on the GPU (bs_render_backward, through the
C-ABI) against the CPU oracle's analytic gradient (oracle/oracle.cpp
render_backward, itself pinned by finite differences of the reference
forward in tests/test_backward_oracle.py).

Bar: per gradient field, max |gpu - oracle| <= 2e-4 * max(1, max |oracle|)
(float32 accumulation and float atomics on the GPU vs double in the
oracle; the forward's exact skip / stop decisions are reproduced, so no
pixel changes its committed set)."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

import oracle_lib as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_2412_17378_b200 import _native as N  # noqa: E402
from paper_2412_17378_b200 import api  # noqa: E402

DEV = "cuda"
TOL = 2e-4


def _case(W, H, pw, ph, n, bgfrac, seed, f=None):
    cam = O.make_camera(focal=(f or float(W), f or float(W)), width=W, height=H)
    g3d = O.gen_clustered_scene(n, cam, seed=seed, sigma=0.035, bgfrac=bgfrac)
    g2d = O.project_all(g3d, cam)
    pl, rg = O.bin_tiles(g2d, W, H, pw, ph)
    rng = np.random.default_rng(seed)
    P = W * H
    dc = rng.normal(size=3 * P).astype(np.float32)
    da = rng.normal(size=P).astype(np.float32)
    dd = (0.1 * rng.normal(size=P)).astype(np.float32)
    return g2d, pl, rg, dc, da, dd


def _compare(got: np.ndarray, ref: np.ndarray):
    assert got.shape == ref.shape
    for j, name in enumerate(O.GRAD_FIELDS):
        scale = max(1.0, float(np.abs(ref[:, j]).max(initial=0.0)))
        err = float(np.abs(got[:, j] - ref[:, j]).max(initial=0.0))
        assert err <= TOL * scale, (name, err, scale)


@pytest.mark.parametrize("W,H,pw,ph,n,bgfrac", [(256, 256, 16, 16, 10000, 1.0), (200, 120, 16, 16, 3000, 0.12),
                                                (300, 170, 16, 8, 6000, 0.3), (130, 90, 8, 8, 2000, 0.5)])
def test_backward_matches_oracle(W, H, pw, ph, n, bgfrac):
    bg = (0.1, 0.2, 0.3)
    g2d, pl, rg, dc, da, dd = _case(W, H, pw, ph, n, bgfrac, seed=7)
    ref = O.render_backward(pl, rg, g2d, W, H, pw, ph, bg, dc, da, dd)
    s = api.splats_from_g2d(g2d, DEV)
    b = api.bin_tiles(s, W, H, pw, ph)
    fwd = api.render_forward(3, s, b, W, H, pw, ph, bg)
    g = api.render_backward(s, b, fwd, W, H, pw, ph, torch.from_numpy(dc).to(DEV), torch.from_numpy(da).to(DEV),
                            torch.from_numpy(dd).to(DEV), bg)
    torch.cuda.synchronize()
    _compare(g.as_fields()[: len(g2d)].double().cpu().numpy(), ref)


def test_backward_super_lists_match_tile_lists():
    """The frame pipeline's 2pw x 2ph super-tile lists (membership-filtered)
    give the tile lists' gradients."""
    W, H, pw, ph = 512, 288, 16, 16
    bg = (0.0, 0.0, 0.0)
    g2d, pl, rg, dc, da, dd = _case(W, H, pw, ph, 20000, 0.12, seed=3, f=600.0)
    ref = O.render_backward(pl, rg, g2d, W, H, pw, ph, bg, dc, da, dd)
    s = api.splats_from_g2d(g2d, DEV)
    b = api.bin_tiles(s, W, H, pw, ph)
    fwd = api.render_forward(3, s, b, W, H, pw, ph, bg)
    sb = api.bin_tiles(s, W, H, 2 * pw, 2 * ph)
    T = b.tile_count
    rt = torch.empty(2 * T, dtype=torch.int32, device=DEV)
    N.call("bs_super_tile_ranges", sb.tile_ranges.data_ptr(), W, H, pw, ph, rt.data_ptr(), api._stream(DEV))
    sup = api.DeviceBinning(b.tile_cols, b.tile_rows, sb.point_list, rt, sb.k)
    args = (torch.from_numpy(dc).to(DEV), torch.from_numpy(da).to(DEV), torch.from_numpy(dd).to(DEV), bg)
    g = api.render_backward(s, sup, fwd, W, H, pw, ph, *args, super_lists=True)
    torch.cuda.synchronize()
    _compare(g.as_fields()[: len(g2d)].double().cpu().numpy(), ref)


def test_backward_colour_only_and_lpt_order():
    """dL/dalpha, dL/ddepth omitted (NULL = zero) and an LPT task order: the
    colour gradients alone."""
    W, H, pw, ph = 192, 160, 16, 16
    bg = (0.2, 0.2, 0.2)
    g2d, pl, rg, dc, _, _ = _case(W, H, pw, ph, 4000, 0.2, seed=11)
    P = W * H
    ref = O.render_backward(pl, rg, g2d, W, H, pw, ph, bg, dc, np.zeros(P, np.float32), np.zeros(P, np.float32))
    s = api.splats_from_g2d(g2d, DEV)
    b = api.bin_tiles(s, W, H, pw, ph)
    st = api.tile_load_histogram(b)
    fwd = api.render_forward(3, s, b, W, H, pw, ph, bg, task_order=st.task_order)
    g = api.render_backward(s, b, fwd, W, H, pw, ph, torch.from_numpy(dc).to(DEV), bg=bg, task_order=st.task_order)
    torch.cuda.synchronize()
    _compare(g.as_fields()[: len(g2d)].double().cpu().numpy(), ref)


def test_backward_errors_and_empty():
    W, H = 64, 64
    s = api.DeviceSplats.empty(1, DEV)
    b = api.DeviceBinning(4, 4, torch.zeros(1, dtype=torch.int32, device=DEV),
                          torch.zeros(32, dtype=torch.int32, device=DEV), 0)
    fwd = api.DeviceFrame.empty(W, H, DEV)
    dc = torch.ones(3 * W * H, device=DEV)
    g = api.render_backward(s, b, fwd, W, H, 16, 16, dc)  # empty lists: nothing accumulates
    torch.cuda.synchronize()
    assert not g.as_fields().any()
    with pytest.raises(N.BsError):
        N.call("bs_render_backward", 7, s.c(), None, b.tile_ranges.data_ptr(), None, W, H, 16, 16,
               (C.c_float * 3)(0, 0, 0), fwd.c(), N.FrameGradIn(dc.data_ptr(), None, None), g.c(), 0, None, 0,
               api._stream(DEV))


@pytest.mark.parametrize("W,H,async_mode,graphs", [(1024, 1024, True, True), (512, 384, False, False),
                                                   (1024, 1024, False, False)])
def test_frame_pipeline_backward_matches_oracle(W, H, async_mode, graphs):
    """bs_context_render_backward on the frame pipeline's last frame (fused
    projection: gradients at the input Gaussian index; super-tile lists at
    >= 1 Mpixel, async K checks and CUDA-graph replays) == the oracle's
    gradient of the same frame, mapped through the visible splats."""
    pw = ph = 16
    n = 20000
    bg = (0.1, 0.2, 0.3)
    cam = O.make_camera(focal=(float(W), float(W)), width=W, height=H)
    g3d = O.gen_clustered_scene(n, cam, seed=5, sigma=0.035, bgfrac=0.2)
    vis = np.array([O.lib().orc_project_gaussian(g3d[i:i + 1].ctypes.data, C.byref(cam),
                                                 np.zeros(1, O.G2D_DTYPE).ctypes.data) for i in range(n)], bool)
    g2d = O.project_all(g3d, cam)
    assert vis.sum() == len(g2d)
    pl, rg = O.bin_tiles(g2d, W, H, pw, ph)
    rng = np.random.default_rng(1)
    P = W * H
    dc = rng.normal(size=3 * P).astype(np.float32)
    da = rng.normal(size=P).astype(np.float32)
    dd = (0.1 * rng.normal(size=P)).astype(np.float32)
    ref = O.render_backward(pl, rg, g2d, W, H, pw, ph, bg, dc, da, dd)
    fp = api.FramePipeline(W, H, pw, ph, DEV, N.ALPHA_EXACT, async_mode=async_mode, graphs=graphs)
    d = api.g3d_to_device(g3d, DEV)
    ncam = N.Camera.from_buffer_copy(bytes(cam))
    for _ in range(3):
        fp.forward(d, n, ncam, variant=3, bg=bg)
    g = fp.backward(n, torch.from_numpy(dc).to(DEV), torch.from_numpy(da).to(DEV), torch.from_numpy(dd).to(DEV))
    torch.cuda.synchronize()
    got = g.as_fields()[:n].double().cpu().numpy()
    assert not got[~vis].any()  # culled Gaussians receive nothing
    _compare(got[vis], ref)
    fp.close()


def test_backward_drives_a_fit():
    """A few gradient-descent steps on the splats' colour and opacity (forward
    and backward on the device, the lists fixed) toward a target frame
    rendered from different colours / opacities: the image loss falls."""
    W, H, pw, ph = 128, 96, 16, 16
    g2d, pl, rg, _, _, _ = _case(W, H, pw, ph, 1500, 0.3, seed=21)
    target = g2d.copy()
    rng = np.random.default_rng(3)
    target["color"] = rng.uniform(0, 1, size=target["color"].shape).astype(np.float32)
    target["opacity"] = np.clip(target["opacity"] * rng.uniform(0.6, 1.2, size=len(target)), 0.05, 0.95)
    bg = (0.0, 0.0, 0.0)
    st = api.splats_from_g2d(target, DEV)
    b = api.bin_tiles(st, W, H, pw, ph)
    tgt = api.render_forward(3, st, b, W, H, pw, ph, bg).color.clone()
    s = api.splats_from_g2d(g2d, DEV)
    losses = []
    for _ in range(15):
        fwd = api.render_forward(3, s, b, W, H, pw, ph, bg)
        diff = fwd.color - tgt
        losses.append(float((diff * diff).sum()))
        g = api.render_backward(s, b, fwd, W, H, pw, ph, 2.0 * diff, bg=bg)
        # normalised steps (the per-splat sums span orders of magnitude)
        gc, go = g.rgbr[:, :3], g.cop[:, 1]
        s.rgbr[:, :3] = (s.rgbr[:, :3] - 0.1 * gc / (gc.abs().max() + 1e-12)).clamp(0.0, 1.0)
        s.cop[:, 1] = (s.cop[:, 1] - 0.05 * go / (go.abs().max() + 1e-12)).clamp(0.02, 0.99)
        # keep power_cut consistent with the opacity: ln(1 / (255 o)) - 0.01
        s.cop[:, 2] = torch.log(1.0 / (255.0 * s.cop[:, 1])) - 0.01
    torch.cuda.synchronize()
    assert losses[-1] < 0.5 * losses[0], losses


@pytest.mark.parametrize("cfg", ["c2", "c4"])
def test_backward_full_size_tile_sampled(cfg):
    """The backward at the headline sizes (C2 1080p/1M, C4 4K/3M): dL/d(planes)
    nonzero only on sampled tiles (the 16 longest lists + 0.3 % random, seed
    42), so the gradients are sums over those tiles' pixels; the GPU runs the
    whole frame on the device binning, the oracle only the sampled tiles on
    the same lists (each checked equal to the reference rule by
    test_gpu_parity)."""
    import bench
    W, H, f, n, bgf, sig = bench.CONFIGS[cfg]
    pw = ph = 16
    bg = (0.1, 0.2, 0.3)
    cam = N.make_camera(None, (f, f), W, H)
    g3d = api.gen_clustered_scene(n, cam, cluster_sigma=sig, background_fraction=bgf)
    pipe = api.Pipeline(W, H, pw, ph, DEV, N.ALPHA_EXACT)
    frame, _ = pipe.forward(api.g3d_to_device(g3d), n, cam, variant=3, bg=bg)
    b, s = pipe.last_binning, pipe.splats
    g2d = api.splats_to_g2d(s)
    cols, rows = (W + pw - 1) // pw, (H + ph - 1) // ph
    T = cols * rows
    rg = b.tile_ranges.cpu().numpy().view(np.uint32)
    lens = (rg[1::2] - rg[0::2]).astype(np.int64)
    rng = np.random.default_rng(42)
    tiles = np.unique(np.concatenate([np.argsort(-lens, kind="stable")[:16], rng.choice(T, T // 300, replace=False)]))
    sub_pl, sub_rg, pos = [], np.zeros(2 * T, np.uint32), 0
    for t in tiles.tolist():
        lst = b.point_list[int(rg[2 * t]):int(rg[2 * t + 1])].cpu().numpy().view(np.uint32)
        sub_rg[2 * t], sub_rg[2 * t + 1] = pos, pos + len(lst)
        sub_pl.append(lst)
        pos += len(lst)
    px = np.zeros((H, W), bool)
    for t in tiles.tolist():
        px[(t // cols) * ph:(t // cols) * ph + ph, (t % cols) * pw:(t % cols) * pw + pw] = True
    m = px.reshape(-1)
    P = W * H
    dc = (rng.normal(size=3 * P).astype(np.float32).reshape(P, 3) * m[:, None]).reshape(-1)
    da = rng.normal(size=P).astype(np.float32) * m
    dd = (0.1 * rng.normal(size=P)).astype(np.float32) * m
    ref = O.render_backward(np.concatenate(sub_pl), sub_rg, g2d, W, H, pw, ph, bg, dc, da, dd)
    assert (ref[:, 6] != 0).sum() > 1000 and (ref[:, 0] != 0).sum() > 1000  # the sample is substantial
    g = api.render_backward(s, b, frame, W, H, pw, ph, torch.from_numpy(dc).to(DEV), torch.from_numpy(da).to(DEV),
                            torch.from_numpy(dd).to(DEV), bg, task_order=pipe.last_stats.task_order)
    torch.cuda.synchronize()
    _compare(g.as_fields()[: len(g2d)].double().cpu().numpy(), ref)
