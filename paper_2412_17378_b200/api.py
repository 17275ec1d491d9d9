"""Python host API over the C-ABI (device memory and streams from PyTorch).

Mirrors the reference's render API (/root/reference/proj/core/include/splatsim):
``project_all`` (preprocess.hpp:59), ``bin_tiles`` (:64-65),
``tile_load_histogram`` (:67), ``render_reference`` (blend.hpp:100-102),
``run_kernel`` (kernels.hpp:104-106), ``variant_name``/``variant_from_name``
(kernels.hpp:25-26) and the selector (adaptive.hpp).  Every compute call goes
through ``lib/libsplatsim_b200.so``; there is no CPU path.  PyTorch only
allocates device memory and supplies the CUDA stream.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N

VARIANTS = N.VARIANTS
ALPHA_EXACT, ALPHA_FAST = N.ALPHA_EXACT, N.ALPHA_FAST


def variant_name(v: int) -> str:
    return N.lib().bs_variant_name(int(v)).decode()


def variant_from_name(name: str):
    v = N.lib().bs_variant_from_name(name.encode())
    return None if v < 0 else v


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _ws(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


@dataclass
class DeviceSplats:
    """Projected splats on the device (bs_splats) + the visible count."""
    xyab: torch.Tensor     # [n_cap, 4] f32
    cop: torch.Tensor      # [n_cap, 4] f32
    rgbr: torch.Tensor     # [n_cap, 4] f32
    n_visible: torch.Tensor  # [1] i32 (device)

    @property
    def n_cap(self) -> int:
        return self.xyab.shape[0]

    def c(self) -> N.Splats:
        return N.Splats(_ptr(self.xyab), _ptr(self.cop), _ptr(self.rgbr))

    @staticmethod
    def empty(n: int, device) -> "DeviceSplats":
        n = max(int(n), 1)
        f = lambda: torch.empty((n, 4), dtype=torch.float32, device=device)  # noqa: E731
        return DeviceSplats(f(), f(), f(), torch.zeros(1, dtype=torch.int32, device=device))


@dataclass
class DeviceBinning:
    """TileBinning on the device (include/splatsim/preprocess.hpp:28-36)."""
    tile_cols: int
    tile_rows: int
    point_list: torch.Tensor   # [K] u32 (stored as int32)
    tile_ranges: torch.Tensor  # [2T] u32 (stored as int32)
    k: int

    @property
    def tile_count(self) -> int:
        return self.tile_cols * self.tile_rows


@dataclass
class DeviceFrame:
    """RenderOutput on the device (include/splatsim/blend.hpp:86-97)."""
    width: int
    height: int
    color: torch.Tensor
    alpha: torch.Tensor
    depth: torch.Tensor
    final_t: torch.Tensor
    contrib: torch.Tensor
    term: torch.Tensor

    @staticmethod
    def empty(width: int, height: int, device) -> "DeviceFrame":
        P = width * height
        f = lambda *s, dt=torch.float32: torch.empty(s, dtype=dt, device=device)  # noqa: E731
        return DeviceFrame(width, height, f(P * 3), f(P), f(P), f(P), f(P, dt=torch.int32), f(P, dt=torch.int32))

    def c(self) -> N.FrameOut:
        return N.FrameOut(_ptr(self.color), _ptr(self.alpha), _ptr(self.depth), _ptr(self.final_t),
                          _ptr(self.contrib), _ptr(self.term))

    def to_numpy(self) -> dict:
        return {k: getattr(self, k).cpu().numpy() for k in ("color", "alpha", "depth", "final_t", "contrib", "term")}


def camera(view=None, focal=(100.0, 100.0), width=0, height=0) -> N.Camera:
    return N.make_camera(view, focal, width, height)


def gen_clustered_scene(n: int, cam: N.Camera, n_clusters: int = 4, seed: int = 42, cluster_sigma: float = 0.035,
                        background_fraction: float = 0.12) -> np.ndarray:
    """Host scene synthesis (src/workload.cpp:198-246) -> structured G3D array."""
    out = np.zeros(int(n), dtype=N.G3D_DTYPE)
    N.call("bs_host_gen_clustered_scene", int(n), int(n_clusters), int(seed), float(cluster_sigma),
           float(background_fraction), C.byref(cam), out.ctypes.data if n else None)
    return out


def g3d_to_device(g3d: np.ndarray, device="cuda") -> torch.Tensor:
    arr = np.ascontiguousarray(g3d).view(np.uint8).reshape(-1)
    return torch.from_numpy(arr.copy()).to(device)


# ---------------------------------------------------------------------------
def project_all(g3d_dev: torch.Tensor, n: int, cam: N.Camera, out: DeviceSplats | None = None,
                ws: torch.Tensor | None = None) -> DeviceSplats:
    """P1-P4 (src/preprocess.cpp:17-64) on the device."""
    dev = g3d_dev.device
    out = out or DeviceSplats.empty(n, dev)
    nbytes = N.lib().bs_preprocess_workspace_bytes(int(n))
    if ws is None or ws.numel() < nbytes:
        ws = _ws(nbytes, dev)
    N.call("bs_preprocess", _ptr(g3d_dev), int(n), C.byref(cam), out.c(), _ptr(out.n_visible), _ptr(ws),
           ws.numel(), _stream(dev))
    return out


def splats_from_g2d(g2d: np.ndarray, device="cuda") -> DeviceSplats:
    n = len(g2d)
    buf = torch.from_numpy(np.ascontiguousarray(g2d).view(np.uint8).reshape(-1).copy()).to(device)
    out = DeviceSplats.empty(n, device)
    N.call("bs_splats_from_g2d", _ptr(buf) if n else None, n, out.c(), _stream(device))
    out.n_visible.fill_(n)
    torch.cuda.current_stream(device).synchronize()
    return out


def splats_to_g2d(s: DeviceSplats) -> np.ndarray:
    n = int(s.n_visible.item())
    buf = torch.empty(max(n, 1) * 44, dtype=torch.uint8, device=s.xyab.device)
    if n:
        N.call("bs_splats_to_g2d", s.c(), n, _ptr(buf), _stream(s.xyab.device))
    return buf[: n * 44].cpu().numpy().view(N.G2D_DTYPE).copy()


class Binner:
    """bin_tiles (src/preprocess.cpp:66-115): count -> K readback -> sort."""

    def __init__(self, width: int, height: int, pw: int, ph: int, device="cuda"):
        self.W, self.H, self.pw, self.ph, self.device = width, height, pw, ph, device
        self.cols = (width + pw - 1) // pw
        self.rows = (height + ph - 1) // ph
        self.ws = None
        self.ws_k = -1
        self.ws_n = -1
        self.k_dev = torch.zeros(1, dtype=torch.int64, device=device)
        self.k_host = torch.zeros(1, dtype=torch.int64, pin_memory=True)
        self.point_list = None
        self.tile_ranges = torch.empty(2 * self.cols * self.rows, dtype=torch.int32, device=device)

    def _ensure_ws(self, n_cap: int, k_cap: int):
        if self.ws is None or n_cap > self.ws_n or k_cap > self.ws_k:
            self.ws_n, self.ws_k = max(n_cap, self.ws_n), max(k_cap, self.ws_k)
            nb = N.lib().bs_bin_workspace_bytes(self.ws_n, self.W, self.H, self.pw, self.ph, self.ws_k)
            self.ws = _ws(nb, self.device)

    def count(self, s: DeviceSplats) -> None:
        self._ensure_ws(s.n_cap, max(self.ws_k, 0))
        N.call("bs_bin_count", s.c(), s.n_cap, _ptr(s.n_visible), self.W, self.H, self.pw, self.ph,
               _ptr(self.k_dev), _ptr(self.ws), self.ws.numel(), _stream(self.device))

    def read_k(self) -> int:
        self.k_host.copy_(self.k_dev, non_blocking=True)
        torch.cuda.current_stream(self.device).synchronize()
        return int(self.k_host.item())

    def sort(self, s: DeviceSplats, k: int) -> DeviceBinning:
        if k > self.ws_k:
            # grow (re-count into the larger workspace: the count state lives in it)
            self._ensure_ws(s.n_cap, int(k * 1.25) + 1024)
            self.count(s)
        if self.point_list is None or self.point_list.numel() < max(k, 1):
            self.point_list = torch.empty(max(int(k * 1.25), 1024), dtype=torch.int32, device=self.device)
        N.call("bs_bin_sort", s.c(), s.n_cap, _ptr(s.n_visible), self.W, self.H, self.pw, self.ph, int(k),
               _ptr(self.point_list), _ptr(self.tile_ranges), _ptr(self.ws), self.ws.numel(), _stream(self.device))
        return DeviceBinning(self.cols, self.rows, self.point_list[:k], self.tile_ranges, k)

    def __call__(self, s: DeviceSplats) -> DeviceBinning:
        self.count(s)
        return self.sort(s, self.read_k())


def bin_tiles(s: DeviceSplats, width: int, height: int, pw: int, ph: int) -> DeviceBinning:
    return Binner(width, height, pw, ph, s.xyab.device)(s)


@dataclass
class TileStats:
    hist: torch.Tensor        # raw bs_tile_histogram bytes (device)
    counts: torch.Tensor      # [T] u32 (int32 storage)
    task_order: torch.Tensor  # [T] LPT order

    def summary(self) -> dict:
        raw = self.hist.cpu().numpy().tobytes()
        h = N.TileHistogram.from_buffer_copy(raw[: C.sizeof(N.TileHistogram)])
        return {"min": h.min, "max": h.max, "p50": h.p50, "p99": h.p99, "mean": h.mean, "total": h.total,
                "tiles": h.tiles, "nonempty": h.nonempty}

    def c_struct(self) -> N.TileHistogram:
        raw = self.hist.cpu().numpy().tobytes()
        return N.TileHistogram.from_buffer_copy(raw[: C.sizeof(N.TileHistogram)])


def tile_load_histogram(b: DeviceBinning, ws: torch.Tensor | None = None) -> TileStats:
    """P6 (src/preprocess.cpp:117-136) + LPT order, on the device."""
    dev = b.tile_ranges.device
    T = b.tile_count
    nb = N.lib().bs_tile_stats_workspace_bytes(T)
    if ws is None or ws.numel() < nb:
        ws = _ws(nb, dev)
    st = TileStats(torch.zeros(64, dtype=torch.uint8, device=dev), torch.empty(max(T, 1), dtype=torch.int32, device=dev),
                   torch.empty(max(T, 1), dtype=torch.int32, device=dev))
    N.call("bs_tile_stats", _ptr(b.tile_ranges), T, _ptr(st.hist), _ptr(st.counts), _ptr(st.task_order), _ptr(ws),
           ws.numel(), _stream(dev))
    return st


def select_variant(stats: TileStats, width: int, height: int, pw: int, ph: int, sm_count: int = 0) -> int:
    h = stats.c_struct()
    v = N.lib().bs_select_variant(C.byref(h), width, height, pw, ph, sm_count)
    N.check("bs_select_variant", 0 if v >= 0 else v)
    return v


def render_workspace(width: int, height: int, device) -> torch.Tensor:
    """The render's workspace (work-queue counters + FineGrainedCombined tail
    hand-off slots).  A workspace belongs to ONE stream at a time: two renders
    sharing one concurrently would race on the queue."""
    return _ws(N.lib().bs_render_workspace_bytes(width, height), device)


def render_forward(variant: int, s: DeviceSplats, b: DeviceBinning, width: int, height: int, pw: int, ph: int,
                   bg=(0.0, 0.0, 0.0), alpha_mode: int = ALPHA_EXACT, task_order: torch.Tensor | None = None,
                   out: DeviceFrame | None = None, ws: torch.Tensor | None = None) -> DeviceFrame:
    """run_kernel(variant, ...) output (src/kernels.cpp:268-301) on the device.

    ``ws``: a caller-owned render workspace (``render_workspace``), reused
    across calls on one stream; without it each call takes a fresh one from
    torch's stream-aware caching allocator."""
    dev = s.xyab.device
    if b.tile_cols != (width + pw - 1) // pw or b.tile_rows != (height + ph - 1) // ph:
        raise ValueError("run_kernel: binning grid does not match image dims")
    out = out or DeviceFrame.empty(width, height, dev)
    need = N.lib().bs_render_workspace_bytes(width, height)
    if ws is None or ws.numel() < need:
        ws = _ws(need, dev)
    bgc = (C.c_float * 3)(*[float(x) for x in bg])
    N.call("bs_render_forward", int(variant), int(alpha_mode), s.c(), _ptr(b.point_list) if b.k else None,
           _ptr(b.tile_ranges), _ptr(task_order), width, height, pw, ph, bgc, out.c(), _ptr(ws), ws.numel(),
           _stream(dev))
    return out


GRAD_FIELDS = ("x", "y", "conic_a", "conic_b", "conic_c", "opacity", "r", "g", "b", "depth")


@dataclass
class SplatGrads:
    """Per-splat gradients in the DeviceSplats layout (bs_splat_grads)."""
    xyab: torch.Tensor  # [n, 4]: d/dx, d/dy, d/dconic_a, d/dconic_b
    cop: torch.Tensor   # [n, 4]: d/dconic_c, d/dopacity, 0, d/ddepth
    rgbr: torch.Tensor  # [n, 4]: d/dr, d/dg, d/db, 0

    @staticmethod
    def zeros(n: int, device) -> "SplatGrads":
        f = lambda: torch.zeros((max(int(n), 1), 4), dtype=torch.float32, device=device)  # noqa: E731
        return SplatGrads(f(), f(), f())

    def c(self) -> N.SplatGrads:
        return N.SplatGrads(_ptr(self.xyab), _ptr(self.cop), _ptr(self.rgbr))

    def as_fields(self) -> torch.Tensor:
        """[n, 10] in GRAD_FIELDS order (the oracle's layout)."""
        x, c, r = self.xyab, self.cop, self.rgbr
        return torch.stack([x[:, 0], x[:, 1], x[:, 2], x[:, 3], c[:, 0], c[:, 1], r[:, 0], r[:, 1], r[:, 2],
                            c[:, 3]], dim=1)


def render_backward(s: DeviceSplats, b: DeviceBinning, fwd: DeviceFrame, width: int, height: int, pw: int, ph: int,
                    dl_dcolor: torch.Tensor, dl_dalpha: torch.Tensor | None = None,
                    dl_ddepth: torch.Tensor | None = None, bg=(0.0, 0.0, 0.0), alpha_mode: int = ALPHA_EXACT,
                    task_order: torch.Tensor | None = None, grads: SplatGrads | None = None,
                    ws: torch.Tensor | None = None, super_lists: bool = False) -> SplatGrads:
    """Backward render: per-splat gradients of the frame
    ``fwd`` (the forward's outputs on the same splats and binning) for the
    given dL/d(colour, alpha, depth); accumulated into ``grads``."""
    dev = s.xyab.device
    if b.tile_cols != (width + pw - 1) // pw or b.tile_rows != (height + ph - 1) // ph:
        raise ValueError("render_backward: binning grid does not match image dims")
    grads = grads or SplatGrads.zeros(s.n_cap, dev)
    if ws is None:
        ws = _ws(256, dev)
    bgc = (C.c_float * 3)(*[float(x) for x in bg])
    dc = dl_dcolor.contiguous()
    da = None if dl_dalpha is None else dl_dalpha.contiguous()
    dd = None if dl_ddepth is None else dl_ddepth.contiguous()
    gin = N.FrameGradIn(_ptr(dc), _ptr(da), _ptr(dd))
    N.call("bs_render_backward", int(alpha_mode), s.c(), _ptr(b.point_list) if b.k else None, _ptr(b.tile_ranges),
           _ptr(task_order), width, height, pw, ph, bgc, fwd.c(), gin, grads.c(), int(super_lists), _ptr(ws),
           ws.numel(), _stream(dev))
    return grads


def frame_work(f: DeviceFrame, b: DeviceBinning, pw: int, ph: int) -> tuple[int, int]:
    """(evaluated, committed) pair counts: E = sum consumed, C = sum contrib."""
    dev = f.color.device
    buf = torch.zeros(2, dtype=torch.int64, device=dev)
    N.call("bs_frame_work", _ptr(f.term), _ptr(f.contrib), _ptr(b.tile_ranges), f.width, f.height, pw, ph,
           _ptr(buf), _stream(dev))
    e, c = buf.cpu().tolist()
    return int(e), int(c)


def sm_count() -> int:
    v = C.c_int32(0)
    N.call("bs_device_sm_count", C.byref(v))
    return int(v.value)


@dataclass
class Pipeline:
    """Device-resident forward pipeline: preprocess -> bin -> stats -> render.

    Buffers persist across frames (resized on growth); one stream (torch's
    current).  ``forward`` returns the frame and the variant used.
    """
    width: int
    height: int
    pw: int = 16
    ph: int = 16
    device: str = "cuda"
    alpha_mode: int = ALPHA_EXACT
    splats: DeviceSplats | None = None
    binner: Binner | None = None
    frame: DeviceFrame | None = None
    pre_ws: torch.Tensor | None = None
    stats_ws: torch.Tensor | None = None
    render_ws: torch.Tensor | None = None  # this pipeline's own (queue counters are per render stream)
    last_variant: int = -1
    last_k: int = 0
    last_stats: TileStats | None = field(default=None, repr=False)
    last_binning: DeviceBinning | None = field(default=None, repr=False)

    def __post_init__(self):
        self.binner = Binner(self.width, self.height, self.pw, self.ph, self.device)
        self.frame = DeviceFrame.empty(self.width, self.height, self.device)
        self.render_ws = render_workspace(self.width, self.height, self.device)

    def forward(self, g3d_dev: torch.Tensor, n: int, cam: N.Camera, variant="auto", bg=(0.0, 0.0, 0.0),
                stage_events: list | None = None):
        """One frame.  stage_events (optional list) receives (name, cuda.Event)
        marks after each stage for a warm per-stage breakdown."""
        def mark(name):
            if stage_events is not None:
                e = torch.cuda.Event(enable_timing=True)
                e.record()
                stage_events.append((name, e))

        mark("start")
        if self.splats is None or self.splats.n_cap < n:
            self.splats = DeviceSplats.empty(n, self.device)
        if self.pre_ws is None or self.pre_ws.numel() < N.lib().bs_preprocess_workspace_bytes(n):
            self.pre_ws = _ws(N.lib().bs_preprocess_workspace_bytes(n), self.device)
        project_all(g3d_dev, n, cam, self.splats, self.pre_ws)
        mark("preprocess")
        self.binner.count(self.splats)
        mark("bin_count")
        k = self.binner.read_k()
        mark("k_readback")
        b = self.binner.sort(self.splats, k)
        mark("bin_sort")
        T = b.tile_count
        if self.stats_ws is None or self.stats_ws.numel() < N.lib().bs_tile_stats_workspace_bytes(T):
            self.stats_ws = _ws(N.lib().bs_tile_stats_workspace_bytes(T), self.device)
        st = tile_load_histogram(b, self.stats_ws)
        if variant == "auto":
            v = select_variant(st, self.width, self.height, self.pw, self.ph)
        else:
            v = variant if isinstance(variant, int) else variant_from_name(variant)
        mark("stats_select")
        render_forward(v, self.splats, b, self.width, self.height, self.pw, self.ph, bg, self.alpha_mode,
                       st.task_order, self.frame, self.render_ws)
        mark("render")
        self.last_variant, self.last_k, self.last_stats, self.last_binning = v, b.k, st, b
        return self.frame, v


STAGES = ("preprocess", "bin_count", "k_readback", "bin_sort", "stats_select", "render")


class FramePipeline:
    """The whole forward through the native frame context
    (``bs_render_frame_device``): one C-ABI call per frame, stream-ordered on
    torch's current stream, one 8-byte host wait (K) and on-device variant
    selection for ``variant="auto"``.  Outputs land in ``self.frame``."""

    def __init__(self, width: int, height: int, pw: int = 16, ph: int = 16, device="cuda",
                 alpha_mode: int = ALPHA_EXACT, timing: bool = False, async_mode: bool = False,
                 graphs: bool = False, fine_ctas: int = 0):
        self.width, self.height, self.pw, self.ph, self.device = width, height, pw, ph, device
        self.ctx = C.c_void_p()
        N.call("bs_context_create", C.byref(self.ctx), int(alpha_mode))
        N.call("bs_context_set_stream", self.ctx, _stream(device))
        if async_mode:  # no host wait inside a frame; K checked at the next call (bs_context_set_async)
            N.call("bs_context_set_async", self.ctx, 1)
        if graphs:  # replay a captured CUDA graph of the frame (bs_context_set_graphs)
            N.call("bs_context_set_graphs", self.ctx, 1)
        if fine_ctas:  # this context's FineGrainedCombined CTAs per SM (bs_context_set_fine_occupancy)
            N.call("bs_context_set_fine_occupancy", self.ctx, int(fine_ctas))
        if timing:
            N.call("bs_context_enable_timing", self.ctx, 1)
        self.frame = DeviceFrame.empty(width, height, device)

    def forward(self, g3d_dev: torch.Tensor, n: int, cam: N.Camera, variant="auto", bg=(0.0, 0.0, 0.0),
                info: bool = False):
        v = -1 if variant == "auto" else (variant if isinstance(variant, int) else variant_from_name(variant))
        bgc = (C.c_float * 3)(*[float(x) for x in bg])
        fi = N.FrameInfo() if info else None
        N.call("bs_render_frame_device", self.ctx, _ptr(g3d_dev), int(n), C.byref(cam), self.pw, self.ph, int(v), bgc,
               self.frame.c(), C.byref(fi) if info else None)
        self._last_n = int(n)
        return self.frame, fi

    def backward(self, n: int, dl_dcolor: torch.Tensor, dl_dalpha: torch.Tensor | None = None,
                 dl_ddepth: torch.Tensor | None = None, grads: "SplatGrads | None" = None) -> "SplatGrads":
        """Backward render of the last frame (bs_context_render_backward):
        per-Gaussian gradients at the input index (n = the frame's Gaussian
        count), accumulated into ``grads``."""
        if n < getattr(self, "_last_n", 0):
            raise ValueError(f"backward: n={n} is below the last frame's {self._last_n} Gaussians")
        grads = grads or SplatGrads.zeros(n, self.device)
        if grads.xyab.shape[0] < n:
            raise ValueError("backward: grads hold fewer than n splats")
        dc = dl_dcolor.contiguous()
        da = None if dl_dalpha is None else dl_dalpha.contiguous()
        dd = None if dl_ddepth is None else dl_ddepth.contiguous()
        N.call("bs_context_render_backward", self.ctx, N.FrameGradIn(_ptr(dc), _ptr(da), _ptr(dd)), grads.c())
        return grads

    def sync(self) -> int:
        """Finish every pending frame (re-rendering any whose K overflowed the
        point_list capacity); returns the number of such re-renders so far."""
        r = C.c_int64(0)
        N.call("bs_context_sync", self.ctx, C.byref(r))
        return int(r.value)

    def graph_launches(self) -> int:
        v = C.c_int64(0)
        N.call("bs_context_graph_launches", self.ctx, C.byref(v))
        return int(v.value)

    def capacity(self) -> tuple[int, int]:
        """(point_list capacity, times grown) — growth inside a timed run is a stall."""
        cap, g = C.c_int64(0), C.c_int64(0)
        N.call("bs_context_capacity", self.ctx, C.byref(cap), C.byref(g))
        return int(cap.value), int(g.value)

    def last_info(self) -> N.FrameInfo:
        fi = N.FrameInfo()
        N.call("bs_context_last_info", self.ctx, C.byref(fi))
        return fi

    def stage_ms(self) -> dict:
        ms = (C.c_float * len(STAGES))()
        N.call("bs_context_stage_ms", self.ctx, ms, len(STAGES))
        return dict(zip(STAGES, [float(x) for x in ms]))

    def close(self):
        if self.ctx:
            torch.cuda.synchronize(self.device)
            N.call("bs_context_destroy", self.ctx)
            self.ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
