#!/usr/bin/env python
"""bench.py — B200 Balanced-3DGS forward render benchmark (driver contract).

Metric (BASELINE.json): fwd render ms/frame + blends/s (1080p, 1M Gaussians);
views/s at 1/2/4/8 GPU.  One step = one full forward of one 1920x1080 view of
the 1M-Gaussian clustered scene (preprocess -> bin -> tile stats -> per-frame
variant selection -> render) on each GPU.  Views come from a 64-view orbit
(yaw -15..+15 deg about the scene pivot), rank r renders views r, r+N, ...:
weak scaling, no collective on the data path (the only collectives are the
timing barrier / max-over-ranks).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import ctypes as C
import gc
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
NCU_COUNTERS_PATH = os.path.join(ROOT, "profiles", "ncu_counters.json")

CONFIGS = {
    # name: (W, H, focal, N gaussians, bg fraction, cluster sigma)
    "c2": (1920, 1080, 1000.0, 1_000_000, 0.12, 0.035),
    "c1": (256, 256, 256.0, 10_000, 1.0, 0.035),
    "c4": (3840, 2160, 2000.0, 3_000_000, 0.12, 0.035),
}
# the view schedule and the orbit are the product's (paper_2412_17378_b200/
# sharding.py; tests/test_sharding_gloo.py covers them with world-size-2 gloo)
from paper_2412_17378_b200.sharding import N_VIEWS, batch_view_ids, orbit_view, views_for_rank  # noqa: E402


def load_counters() -> dict:
    """Per-kernel ncu counters (one --set full capture of each render kernel
    on each config, tools/ncu_counters.py -> profiles/ncu_counters.json)."""
    try:
        with open(NCU_COUNTERS_PATH) as f:
            return json.load(f)
    except Exception:
        return {}


def load_peaks() -> dict:
    try:
        with open(PEAKS_PATH) as f:
            return json.load(f)
    except Exception:
        return {}


class NvmlClockSampler:
    """SM clock + clock-event reasons sampled in-process through NVML (what
    nvidia-smi reports) during the timed region — no subprocess, so no extra
    driver client polling the GPU while frames run."""

    NAMES = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
             ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
             ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
             ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, gpu_index: int, period_s: float = 0.05):
        self.gpu, self.period = gpu_index, period_s
        self.sm, self.smax, self.reasons = [], None, set()
        self.stop_ev = threading.Event()
        self.t = None

    def start(self):
        import pynvml as nv
        nv.nvmlInit()
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        idx = int(vis.split(",")[self.gpu]) if vis and vis.split(",")[0].strip().isdigit() else self.gpu
        self.nv, self.h = nv, nv.nvmlDeviceGetHandleByIndex(idx)
        self.smax = float(nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM))
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def _run(self):
        nv = self.nv
        while not self.stop_ev.is_set():
            self.sm.append(float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            for name, const in self.NAMES:
                if r & getattr(nv, const):
                    self.reasons.add(name)
            self.stop_ev.wait(self.period)

    def stop(self) -> dict:
        self.stop_ev.set()
        if self.t:
            self.t.join(timeout=2)
        return {"sm_mhz": float(np.median(self.sm)) if self.sm else None, "sm_max_mhz": self.smax,
                "reasons": sorted(self.reasons), "samples": len(self.sm), "source": "nvml"}


class NoClockSampler:
    def stop(self) -> dict:
        return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["sampling disabled (BS_CLOCKS=off)"], "samples": 0}


def make_clock_sampler(gpu_index: int):
    """NVML in-process sampler; nvidia-smi subprocess if NVML is unusable."""
    if os.environ.get("BS_CLOCKS") == "off":
        return NoClockSampler()
    if os.environ.get("BS_CLOCKS", "nvml") == "nvml":
        try:
            s = NvmlClockSampler(gpu_index)
            s.start()
            return s
        except Exception:
            pass
    s = ClockSampler(gpu_index)
    s.start()
    return s


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines: list[str] = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.t:
            self.t.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
def cpu_libs():
    """(oracle port, reference library or None, kind).  The reference itself
    (oracle/_ref: /root/reference's own sources built here against the
    Eigen-subset shim; the built .so travels to the GPU box) when present,
    else the oracle restatement.  Test / baseline infrastructure only."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_lib as O
    try:
        import ref_lib as R
        if os.path.exists(R.REF_LIB):
            R.lib()
            return O, R, "reference"
    except Exception:
        pass
    return O, None, "port"


def cpu_full_frame(O, R, g3d, cam, W, H, pw, ph, variant: int, threads: int) -> dict:
    """One COMPLETE frame on the host: project_all -> bin_tiles -> run_kernel,
    the reference's own functions when R is given (project_all split over
    `threads` contiguous chunks — an order-preserving map; bin_tiles is the
    reference's single-threaded sort; run_kernel over tile sets dealt to
    `threads` threads — tiles are independent, the result is one call's),
    else the oracle port.  Returns per-stage seconds."""
    t0 = time.perf_counter()
    g2d = R.project_all(g3d, cam, threads) if R else O.project_all(g3d, cam)
    t1 = time.perf_counter()
    pl, rg = (R or O).bin_tiles(g2d, W, H, pw, ph)
    t2 = time.perf_counter()
    if R:
        R.run_kernel(variant, pl, rg, g2d, W, H, pw, ph, (0, 0, 0), threads=threads)
    else:
        O.render(variant, pl, rg, g2d, W, H, pw, ph, (0, 0, 0), lazy=False, threads=threads)
    t3 = time.perf_counter()
    return {"project_s": t1 - t0, "bin_s": t2 - t1, "render_s": t3 - t2, "frame_s": t3 - t0,
            "K": int(len(pl)), "n_visible": int(len(g2d))}


def cpu_sample_estimate(O, R, g3d, cam_o, g2d, pl, ranges, W, H, pw, ph, budget_s: float, variant: int = 0,
                        seed: int = 0):
    """Bounded sample of one frame on ONE host thread (the reference has no
    threads), extrapolated to the full frame:
      project_all on 1/8 of the Gaussians        x8 (linear)
      bin_tiles on 1/8 of the projected splats    x K log K ratio
      run_kernel (faithful: evaluates the whole tile list per pixel,
        src/blend.cpp:85-92) on random tiles     x (sum pixels*len) ratio
    through the reference's own code (R) when built, else the oracle port."""
    rng = np.random.default_rng(seed)
    lib = R or O
    n = len(g3d)
    div = 8
    sub = np.sort(rng.choice(n, size=max(1, n // div), replace=False))
    g3s = np.ascontiguousarray(g3d[sub])
    t0 = time.perf_counter()
    R.project_all(g3s, cam_o, 1) if R else O.project_all(g3s, cam_o)
    t_proj = (time.perf_counter() - t0) * (n / len(sub))
    m = len(g2d)
    sub2 = np.sort(rng.choice(m, size=max(1, m // div), replace=False))
    g2s = np.ascontiguousarray(g2d[sub2])
    t0 = time.perf_counter()
    pl_s, _ = lib.bin_tiles(g2s, W, H, pw, ph)
    t_bin_s = time.perf_counter() - t0
    K, Ks = max(len(pl), 2), max(len(pl_s), 2)
    t_bin = t_bin_s * (K * math.log(K)) / (Ks * math.log(Ks))
    cols, rows = (W + pw - 1) // pw, (H + ph - 1) // ph
    lens = (ranges[1::2].astype(np.int64) - ranges[0::2].astype(np.int64))
    tx, ty = np.arange(cols * rows) % cols, np.arange(cols * rows) // cols
    pix = (np.minimum(W, (tx + 1) * pw) - tx * pw) * (np.minimum(H, (ty + 1) * ph) - ty * ph)
    work = pix * lens
    total_work = int(work.sum())
    target = 0.6 * budget_s / 8e-9  # ~8 ns per evaluated pair (order of magnitude)
    order = rng.permutation(cols * rows)
    csum = np.cumsum(work[order])
    cut = int(np.searchsorted(csum, min(target, total_work))) + 1
    tiles = np.sort(order[:cut]).astype(np.int32)
    t0 = time.perf_counter()
    if R:  # the sampled tiles' lists, every other tile empty
        sr = np.zeros_like(ranges)
        sr[2 * tiles], sr[2 * tiles + 1] = ranges[2 * tiles], ranges[2 * tiles + 1]
        R.run_kernel(variant, pl, sr, g2d, W, H, pw, ph, (0, 0, 0), threads=1)
    else:
        O.render(variant, pl, ranges, g2d, W, H, pw, ph, (0, 0, 0), lazy=False, threads=1, tiles=tiles)
    t_r_s = time.perf_counter() - t0
    sw = max(1, int(work[tiles].sum()))
    t_render = t_r_s * total_work / sw
    desc = (f"{'reference (oracle/_ref)' if R else 'oracle port'}, 1 thread: project_all on {len(sub)}/{n} Gaussians "
            f"(x{n / len(sub):.1f}); bin_tiles on {len(sub2)}/{m} splats (x K log K); run_kernel faithful on "
            f"{len(tiles)}/{cols * rows} random tiles ({sw / total_work * 100:.2f}% of pixel*list work, extrapolated)")
    return t_proj + t_bin + t_render, {"project_s": t_proj, "bin_s": t_bin, "render_s": t_render}, desc


# ---------------------------------------------------------------------------
def run_reference(args) -> None:
    """--impl reference: the reference's own CPU implementation of the path
    (oracle/_ref when built, else the oracle port) on the host cores, on
    this arm's workload: every timed step is one COMPLETE view of the C2
    orbit (project_all -> bin_tiles -> run_kernel(FineGrainedCombined), the
    variant our arm's selector runs), all host threads where the reference's
    functions allow it.  Warm-up steps run project_all only (a CPU has no
    JIT or clock ramp to warm; a full warm-up frame would add ~15 s each)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    O, R, kind = cpu_libs()
    W, H, f, n, bgf, sig = CONFIGS[args.config]
    pw = ph = 16
    threads = os.cpu_count() or 1
    cam0 = O.make_camera(orbit_view(0), (f, f), W, H)
    g3d = (R or O).gen_clustered_scene(n, cam0, sigma=sig, bgfrac=bgf)
    cams = [O.make_camera(orbit_view(k), (f, f), W, H) for k in range(N_VIEWS)]
    for i in range(args.warmup):
        R.project_all(g3d, cams[i % N_VIEWS], threads) if R else O.project_all(g3d, cams[i % N_VIEWS])
    stages = []
    t0 = time.perf_counter()
    for i in range(args.steps):
        stages.append(cpu_full_frame(O, R, g3d, cams[i % N_VIEWS], W, H, pw, ph, 3, threads))
    wall = time.perf_counter() - t0
    value = args.steps / wall
    mean = {k: float(np.mean([s[k] for s in stages])) for k in ("project_s", "bin_s", "render_s", "frame_s")}
    sample = (f"{args.steps} complete C2 views (views 0..{args.steps - 1} of the orbit): "
              f"{'the reference itself (oracle/_ref: /root/reference/proj/core/src built against the Eigen-subset shim)' if R else 'oracle port'}"
              f"; project_all on {threads} threads (contiguous chunks), bin_tiles single-threaded (the reference's sort), "
              f"run_kernel(FineGrainedCombined) over tile sets on {threads} threads")
    out = {"impl": "reference", "metric": metric_name(args.config), "value": value, "unit": "views/s",
           "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": wall / args.steps * 1e3,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
           "dtype": "f32+f64 (f32 alpha/T, f64 colour/depth accumulators)",
           "data": "synthetic: gen_clustered_scene seed 42",
           "config": config_desc(args.config, W, H, n, pw, ph),
           "cpu_baseline": {"value": value, "unit": "views/s", "cores": threads, "kind": kind, "sample": sample,
                            "stage_s": mean, "K_mean": float(np.mean([s["K"] for s in stages]))},
           "e2e": {"value": value, "unit": "views/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def auto_streams(W: int, H: int) -> int:
    """Frame contexts for --streams 0: small frames are launch-latency-bound
    (more frames in flight fill the GPU), large ones are render-bound (a
    fifth+ context only adds contention)."""
    return 8 if W * H < (1 << 20) else 4


def metric_name(cfg: str) -> str:
    return "fwd render views/s (1080p, 1M Gaussians; full forward per view)" if cfg == "c2" else \
        f"fwd render views/s ({cfg})"


def config_desc(cfg, W, H, n, pw, ph) -> dict:
    _, _, f, _, bgf, sig = CONFIGS[cfg]
    return {"workload": f"{cfg.upper()}: {W}x{H}, focal {f:g}, {n} Gaussians from gen_clustered_scene (4 clusters, "
                        f"sigma {sig:g}, background fraction {bgf:g}), {pw}x{ph} tiles, views from the 64-view "
                        "+-15 deg yaw orbit",
            "global_batch": None, "seq_len": None}


# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--alpha", default="exact", choices=["exact", "fast"])
    ap.add_argument("--variant", default="auto")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sync-frames", action="store_true", help="wait for K inside each frame (no async mode)")
    ap.add_argument("--no-graphs", action="store_true", help="launch every kernel instead of replaying a CUDA graph")
    ap.add_argument("--streams", type=int, default=0,
                    help="frame contexts on separate streams (views round-robin); 0 = auto: 8 for frames below "
                         "1 Mpixel (launch-latency-bound: C1 12.1k -> 14.5k views/s), else 4 (C2: 8 measured "
                         "7 %% slower)")
    ap.add_argument("--fine-ctas", type=int, default=0,
                    help="FineGrainedCombined CTAs per SM per context when streams > 1 (0 = as many as fit; "
                         "tools/sweep_occupancy.sh: uncapped is best with the r2 kernels)")
    ap.add_argument("--no-extras", action="store_true", help="skip per-variant sweep / e2e / cpu baseline")
    ap.add_argument("--no-c3", action="store_true", help="skip the C3 imbalance sweep in the extras")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--batch", type=int, default=N_VIEWS,
                    help="views per step: the fixed batch of the first B orbit views, split contiguously over the "
                         "ranks (SURVEY 8e, strong scaling); 0 = one view per rank per step (weak scaling)")
    args = ap.parse_args()

    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist

    from paper_2412_17378_b200 import _native as N
    from paper_2412_17378_b200 import api

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # BS_BENCH_SHARED_GPU=1 (test only): every rank on cuda:0 with gloo, so
    # the N>1 path (view sharding, barriers, max over ranks) runs on a 1-GPU box
    shared = os.environ.get("BS_BENCH_SHARED_GPU") == "1"
    gpu = 0 if shared else local
    torch.cuda.set_device(gpu)
    dev = f"cuda:{gpu}"
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device(dev))

    W, H, f, n, bgf, sig = CONFIGS[args.config]
    pw = ph = 16
    mode = N.ALPHA_EXACT if args.alpha == "exact" else N.ALPHA_FAST
    variant = args.variant if args.variant == "auto" else api.variant_from_name(args.variant)

    cam0 = api.camera(orbit_view(0), (f, f), W, H)
    g3d = api.gen_clustered_scene(n, cam0, cluster_sigma=sig, background_fraction=bgf)
    g3d_dev = api.g3d_to_device(g3d, dev)  # scene replica, uploaded once (outside timing)
    cams = [api.camera(orbit_view(k), (f, f), W, H) for k in range(N_VIEWS)]
    # the native frame pipeline: one C-ABI call per view, no host wait inside a
    # frame (async mode: K verified two calls later, overflowed frames
    # re-rendered), CUDA-graph replay; --streams contexts on their own streams
    # take the views round-robin, so view i+1's preprocess / binning overlaps
    # view i's render
    ns = max(1, args.streams) if args.streams > 0 else auto_streams(W, H)
    args.streams = ns
    fine_ctas = args.fine_ctas if ns > 1 else 0  # leave SM room for the other contexts' kernels during a render
    streams = [torch.cuda.Stream(device=dev) for _ in range(ns)]
    fps = []
    for s_ in streams:
        with torch.cuda.stream(s_):
            fps.append(api.FramePipeline(W, H, pw, ph, dev, mode, async_mode=not args.sync_frames,
                                         graphs=not (args.sync_frames or args.no_graphs), fine_ctas=fine_ctas))
    fp = fps[0]
    # one L2 flush (256 MiB write > 126 MB L2) per step on the step's stream,
    # INSIDE the timed region (conservative: its time counts)
    flushes = [torch.empty(256 << 20, dtype=torch.uint8, device=dev) for _ in range(ns)]

    # every step renders the same fixed batch of args.batch views,
    # split contiguously over the ranks (sharding.batch_view_ids); --batch 0:
    # one view per rank per step, round-robin over the orbit (views_for_rank)
    batch = max(0, args.batch)
    per_step = len(batch_view_ids(rank, world, 1, batch)) if batch else 1

    def view_ids(first_step, steps):
        if batch:
            return batch_view_ids(rank, world, steps, batch)
        return views_for_rank(rank, world, first_step + steps)[first_step:]

    # the whole batch of views is enqueued by one native call
    # (bs_render_views: view i on context i % ns, its L2 flush first), so the
    # host-side cost per view is the C++ loop's, not the interpreter's
    ctx_arr = (C.c_void_p * ns)(*[f_.ctx.value for f_ in fps])
    flush_arr = (C.c_void_p * ns)(*[t_.data_ptr() for t_ in flushes])
    cam_arr = (N.Camera * N_VIEWS)(*cams)
    v_int = -1 if variant == "auto" else int(variant)
    bg_arr = (C.c_float * 3)(0.0, 0.0, 0.0)

    def run_views(first_step, steps, flush=True):
        vids = view_ids(first_step, steps)
        ids = (C.c_int32 * max(1, len(vids)))(*vids)
        N.call("bs_render_views", ctx_arr, ns, C.c_void_p(g3d_dev.data_ptr()), int(n), cam_arr, ids, len(vids), pw, ph,
               v_int, bg_arr, flush_arr if flush else None, (256 << 20) if flush else 0)
        return vids

    def sync_all() -> int:
        return sum(f.sync() for f in fps)

    clk = make_clock_sampler(gpu)  # sampling spans warm-up + timed region (the timed region alone is < 1 s)
    # >= 2 frames per context: capacity calibrated, graphs captured
    run_views(0, max(args.warmup, -(-2 * ns // per_step)), flush=False)
    sync_all()
    torch.cuda.synchronize()

    used = {}
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    reruns_warm = sync_all()
    grows_warm = sum(f.capacity()[1] for f in fps)
    glaunch0 = sum(f.graph_launches() for f in fps)
    launches0 = N.lib().bs_kernel_launches()
    main = torch.cuda.current_stream(dev)
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    gc.disable()  # no collector pauses while the host enqueues the timed frames
    t_start.record(main)
    for s_ in streams:
        s_.wait_stream(main)
    timed_views = run_views(args.warmup, args.steps)
    for s_ in streams:  # join: the end event follows every context's last frame
        main.wait_stream(s_)
    t_end.record(main)
    reruns = sync_all() - reruns_warm  # a re-render would land before the sync point
    gc.enable()
    torch.cuda.synchronize()
    launches = int(N.lib().bs_kernel_launches() - launches0)
    grows = sum(f.capacity()[1] for f in fps) - grows_warm
    graph_replays = sum(f.graph_launches() for f in fps) - glaunch0
    # which variant the on-device selector picked for each timed view (replayed untimed)
    for vid in sorted(set(timed_views)):
        _, fi = fp.forward(g3d_dev, n, cams[vid], variant=variant, info=True)
        used[fi.variant] = used.get(fi.variant, 0) + 1
    if world > 1:
        dist.barrier()
    clocks = clk.stop()
    total_ms = t_start.elapsed_time(t_end)
    if reruns:  # re-renders were enqueued after t_end: time them into the run
        total_ms *= 1.0 + reruns / max(1, len(timed_views))
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        if shared:
            t = t.cpu()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_ms = float(t.item())
    views_per_step = batch if batch else world  # all ranks
    value = views_per_step * args.steps / (max_ms / 1e3)

    extras = {}
    if rank == 0 and not args.no_extras:
        extras = rank0_extras(args, api, N, torch, g3d, g3d_dev, cams, fp, W, H, pw, ph, n, mode, dev, world)

    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank != 0:
        return
    out = {
        "metric": metric_name(args.config),
        "value": value,
        "unit": "views/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": max_ms / args.steps,
        "higher_is_better": True,
        "scaling": "strong" if batch else "weak",
        "vs_baseline": None,
        "views_per_step": views_per_step,
        "dtype": "f32+f64 (f32 alpha/T, f64 colour/depth accumulators)" if mode == N.ALPHA_EXACT else "f32",
        "data": "synthetic: gen_clustered_scene seed 42 (no dataset)",
        "config": dict(config_desc(args.config, W, H, n, pw, ph), alpha_mode=args.alpha, variant=args.variant,
                       variants_used={api.variant_name(k): c for k, c in used.items()},
                       parallelism=(f"view-sharded x{world}: each step is the fixed batch of orbit views 0..{batch - 1}, "
                                    f"split contiguously ({per_step} per rank); scene replicated, no data-path "
                                    f"collective" if batch else
                                    f"view-sharded x{world}: one view per rank per step, round-robin over the "
                                    f"orbit; scene replicated, no data-path collective"),
                       l2="flushed before every step (256 MiB write on the step's stream, inside the timed region)",
                       streams=ns, fine_ctas_per_sm=(args.fine_ctas or "max") if ns > 1 else "max"),
        "gpu_launches": launches,
        "async_reruns": reruns,
        "point_list_grows": grows,
        "graph_replays": graph_replays,
        "clocks": clocks,
    }
    out.update(extras)
    print(json.dumps(out), flush=True)


C3_POINTS = [(1.0, 0.035), (0.8, 0.032), (0.6, 0.03), (0.4, 0.027), (0.25, 0.025), (0.12, 0.022), (0.05, 0.02)]


def c3_sweep(api, N, torch, W, H, pw, ph, n, f, mode, dev) -> dict:
    """SURVEY 8d C3 on the C2 geometry: background_fraction 1.0 -> 0.05 with
    cluster_sigma 0.035 -> 0.02 (uniform -> clustered).  Per point: warm
    render times (CUDA events, median of 5) of every variant on the point's
    16x16 TileBinning, the balanced kernels' ratio to the pixel-wise
    baseline, the device selector's choice and its regret
    t(chosen) / min_v t(v) - 1."""
    out = {"points": []}
    stream = torch.cuda.current_stream()
    cam = api.camera(np.eye(4, dtype=np.float32), (f, f), W, H)
    for bgf, sig in C3_POINTS:
        g3d = api.gen_clustered_scene(n, cam, cluster_sigma=sig, background_fraction=bgf)
        pipe = api.Pipeline(W, H, pw, ph, dev, mode)
        frame, v_auto = pipe.forward(api.g3d_to_device(g3d, dev), n, cam, variant="auto")
        s, b, st = pipe.splats, pipe.last_binning, pipe.last_stats
        ms = {}
        for v in range(5):
            api.render_forward(v, s, b, W, H, pw, ph, (0, 0, 0), mode, st.task_order, frame, pipe.render_ws)
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(5)]
            for a, e in ev:
                a.record(stream)
                api.render_forward(v, s, b, W, H, pw, ph, (0, 0, 0), mode, st.task_order, frame, pipe.render_ws)
                e.record(stream)
            torch.cuda.synchronize()
            ms[api.variant_name(v)] = round(float(np.median([a.elapsed_time(e) for a, e in ev])), 4)
        summ = st.summary()
        best = min(ms.values())
        out["points"].append({
            "background_fraction": bgf, "cluster_sigma": sig, "K": b.k, "tile_max": summ["max"],
            "tile_mean": round(summ["mean"], 1), "render_ms": ms,
            "fg_over_naive": round(ms["Naive"] / ms["FineGrainedCombined"], 3),
            "gw_over_naive": round(ms["Naive"] / ms["GaussianWise"], 3),
            "selected": api.variant_name(v_auto), "regret": round(ms[api.variant_name(v_auto)] / best - 1.0, 4)})
        del pipe, frame, s, b, st
        torch.cuda.empty_cache()
    ext = max(out["points"], key=lambda p: p["tile_max"] / max(1.0, p["tile_mean"]))
    out["most_imbalanced"] = {"background_fraction": ext["background_fraction"], "cluster_sigma": ext["cluster_sigma"],
                              "fg_over_naive": ext["fg_over_naive"], "gw_over_naive": ext["gw_over_naive"],
                              "north_star_target": 3.0}
    out["def"] = ("render-kernel times on each point's 16x16 TileBinning (bs_render_forward), warm, one identity view "
                  "of the C2 geometry; most_imbalanced = the point with the largest max/mean tile list length")
    return out


def rank0_extras(args, api, N, torch, g3d, g3d_dev, cams, fp, W, H, pw, ph, n, mode, dev, world) -> dict:
    res = {}
    peaks = load_peaks()
    # warm per-stage breakdown of the full forward (CUDA events between the
    # native pipeline's stages)
    stage_ms = {}
    reps = 20
    N.call("bs_context_enable_timing", fp.ctx, 1)
    vsel_arg = "auto" if args.variant == "auto" else api.variant_from_name(args.variant)
    for i in range(reps):
        fp.forward(g3d_dev, n, cams[i % N_VIEWS], variant=vsel_arg)
        for k, v in fp.stage_ms().items():
            stage_ms[k] = stage_ms.get(k, 0.0) + v / reps
    N.call("bs_context_enable_timing", fp.ctx, 0)
    res["stage_ms"] = {k: round(v, 4) for k, v in stage_ms.items()}
    pipe = api.Pipeline(W, H, pw, ph, dev, mode)  # stage-by-stage pipeline: keeps splats / binning for the sweeps
    cam_id = api.camera(np.eye(4, dtype=np.float32), cams[0].focal, W, H)  # C2 identity view
    frame, v_auto = pipe.forward(g3d_dev, n, cam_id, variant="auto")
    s, b, st = pipe.splats, pipe.last_binning, pipe.last_stats
    summ = st.summary()
    stream = torch.cuda.current_stream()

    def time_render(variant, m, reps=5):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        api.render_forward(variant, s, b, W, H, pw, ph, (0, 0, 0), m, st.task_order, frame, pipe.render_ws)
        for a, e in ev:
            a.record(stream)
            api.render_forward(variant, s, b, W, H, pw, ph, (0, 0, 0), m, st.task_order, frame, pipe.render_ws)
            e.record(stream)
        torch.cuda.synchronize()
        return float(np.mean([a.elapsed_time(e) for a, e in ev]))

    per_variant = {}
    for m, mname in ((N.ALPHA_EXACT, "exact"), (N.ALPHA_FAST, "fast")):
        per_variant[mname] = {api.variant_name(v): round(time_render(v, m), 4) for v in range(5)}
    mname = "exact" if mode == N.ALPHA_EXACT else "fast"
    vsel = v_auto if args.variant == "auto" else api.variant_from_name(args.variant)
    t_render = time_render(vsel, mode, reps=10)
    api.render_forward(vsel, s, b, W, H, pw, ph, (0, 0, 0), mode, st.task_order, frame, pipe.render_ws)
    E, Cc = api.frame_work(frame, b, pw, ph)
    K, P = b.k, W * H
    ops = 16 * E + 8 * Cc
    fp32_peak = 148 * 128 * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    mufu_peak = 148 * 16 * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    hbm_src = "of measured (MEASURED_PEAKS.json hbm_gbs)" if "hbm_gbs" in peaks else \
        "of fallback (B200_PROFILING.md: 6.65 TB/s, MEASURED_PEAKS.json absent)"
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0)) * 1e9
    bytes_alg = 44 * K + 32 * P
    t_s = t_render / 1e3
    t_roof = max(ops / fp32_peak, E / mufu_peak, bytes_alg / hbm_peak)
    traffic = (load_counters().get(f"{args.config}_{api.variant_name(vsel)}_{mname}") or {}).get("dram_bytes")
    res["fwd_render_ms_per_frame"] = t_render
    res["blends_per_s"] = E / t_s
    res["frame_work"] = {"evaluated_pairs_E": E, "committed_pairs_C": Cc, "tile_instances_K": K, "pixels": P,
                         "tile_stats": summ, "variant": api.variant_name(vsel)}
    res["render_ms_by_variant"] = per_variant
    # SURVEY 8f(4) backward render (the training step's next kernel): per-splat
    # gradients of this frame (exact mode, FineGrainedCombined schedule) for a
    # synthetic dL/d(colour, alpha, depth); kernel time, warm, grads zeroed
    # outside the events
    gen = torch.Generator(device=dev)
    gen.manual_seed(0)
    dl = [torch.randn(k * P_, device=dev, generator=gen) for k, P_ in ((3, W * H), (1, W * H), (1, W * H))]
    api.render_forward(3, s, b, W, H, pw, ph, (0, 0, 0), N.ALPHA_EXACT, st.task_order, frame, pipe.render_ws)
    grads = api.SplatGrads.zeros(s.n_cap, dev)
    bt = []
    for _ in range(6):
        for t_ in (grads.xyab, grads.cop, grads.rgbr):
            t_.zero_()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        api.render_backward(s, b, frame, W, H, pw, ph, dl[0], dl[1], dl[2], (0, 0, 0), N.ALPHA_EXACT, st.task_order,
                            grads, pipe.render_ws)
        e.record(stream)
        torch.cuda.synchronize()
        bt.append(a.elapsed_time(e))
    res["bwd_render_ms_per_frame"] = round(float(np.median(bt[1:])), 4)
    res["bwd_def"] = ("bs_render_backward on the C2 identity view's 16x16 lists: dL/d(x, y, conic, opacity, rgb, "
                      "depth) per splat for random dL/d(colour, alpha, depth); the forward's decisions replayed "
                      "(exact alpha), 10 gradient terms per committed pair warp-reduced, float atomics")
    del grads, dl
    naive = per_variant[mname]["Naive"]
    res["speedup_vs_naive"] = {k: round(naive / v, 3) for k, v in per_variant[mname].items()}
    # list entries any pixel of a tile still reads under the serial semantics:
    # the tile's longest consumed prefix (max over its pixels of term, or the
    # whole list) — K*44 over-counts lists whose tail lies past every stop
    term = frame.term.cpu().numpy().reshape(H, W)
    rg = b.tile_ranges.cpu().numpy().view(np.uint32)
    cols, rows = (W + pw - 1) // pw, (H + ph - 1) // ph
    lens = (rg[1::2].astype(np.int64) - rg[0::2].astype(np.int64)).reshape(rows, cols)
    cons = np.where(term > 0, term, np.repeat(np.repeat(lens, ph, 0), pw, 1)[:H, :W]).astype(np.int64)
    pad = np.zeros((rows * ph, cols * pw), np.int64)
    pad[:H, :W] = cons
    prefix_entries = int(pad.reshape(rows, ph, cols, pw).max(axis=(1, 3)).sum())
    bytes_prefix = 44 * prefix_entries + 32 * P
    # the consumed-work histogram beside the list-length one
    # (consumed(p) = term > 0 ? term : list length, src/kernels.cpp:296)
    qs = (50, 90, 99, 99.9, 100)
    res["frame_work"]["consumed_per_pixel"] = {f"p{q:g}": int(np.percentile(cons, q)) for q in qs}
    res["frame_work"]["consumed_per_pixel"]["mean"] = round(float(cons.mean()), 1)
    res["frame_work"]["list_len_per_tile"] = {f"p{q:g}": int(np.percentile(lens, q)) for q in qs}
    # the render the timed frames run: on >= 1 Mpixel frames the frame
    # pipeline bins into 2pw x 2ph super-tile lists and the render filters
    # each tile's members (bs_render_forward_super) — time that render stage
    # (CUDA events on the frame's stream) on the same view
    N.call("bs_context_enable_timing", fp.ctx, 1)
    t_fp = []
    for _ in range(10):
        fp.forward(g3d_dev, n, cam_id, variant=vsel_arg)
        t_fp.append(fp.stage_ms()["render"])
    N.call("bs_context_enable_timing", fp.ctx, 0)
    sup = C.c_int32(0)
    N.call("bs_context_list_mode", fp.ctx, C.byref(sup))
    t_api_s = t_s
    if sup.value:
        t_s = float(np.mean(t_fp)) / 1e3
    # the lower bound: SURVEY 8d's terms with the HBM term over the bytes
    # blending must read (the consumed list prefixes); the formula as
    # written (44 B per tile instance K) is reported beside it — it exceeds
    # the measured time when list tails lie past every pixel's stop (C4)
    t_roof_survey = t_roof
    t_roof = max(ops / fp32_peak, E / mufu_peak, bytes_prefix / hbm_peak)
    api_view = {"kernel": f"render {api.variant_name(vsel)} ({mname}) on the reference's pw x ph TileBinning "
                          "(bs_render_forward, the API path)", "t_ms": t_api_s * 1e3,
                "frac": ops / t_api_s / fp32_peak, "t_roof_frac": t_roof / t_api_s, "traffic": traffic}
    if sup.value:
        traffic = (load_counters().get(f"{args.config}_{api.variant_name(vsel)}_{mname}_super") or {}).get(
            "dram_bytes")
    res["fwd_render_ms_per_frame_pipeline"] = t_s * 1e3
    kname = (f"render {api.variant_name(vsel)} ({mname}) on super-tile lists (frame pipeline: the timed frames' "
             "render stage)") if sup.value else f"render {api.variant_name(vsel)} ({mname})"
    # The bound is chosen from MEASURED counters of this kernel (one ncu
    # --set full capture per change, profiles/ncu_counters.json, written by
    # tools/ncu_counters.py): the time its measured warp instructions need at
    # one issue per scheduler per clock (148 SMs x 4) vs the time its
    # consumed-prefix bytes (what tile-serial blending must read) and its
    # measured DRAM bytes need at the HBM peak.  The headline achieved / peak
    # / frac is then the ALGORITHMIC work of that resource (SURVEY 8d:
    # 16E + 8C FP32-pipe instructions, or 44K + 32P bytes) per launch over the
    # measured launch time.
    ckey = f"{args.config}_{api.variant_name(vsel)}_{mname}" + ("_super" if sup.value else "")
    cnt = load_counters().get(ckey)
    clk_hz = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    issue_peak = 148 * 4 * clk_hz  # warp instructions / s
    measured = {}
    if cnt:
        measured = {"counters_key": ckey, "source": cnt.get("source"),
                    "warp_instructions": cnt.get("inst_executed"), "dram_bytes": cnt.get("dram_bytes"),
                    "issue_slot_util_ncu": cnt.get("issue_active_pct")}
        if cnt.get("inst_executed"):
            measured["t_issue_ms"] = cnt["inst_executed"] / issue_peak * 1e3
            measured["issue_util"] = cnt["inst_executed"] / issue_peak / t_s
            measured["thread_instr_per_evaluated_pair"] = (cnt["inst_executed"] * cnt.get("avg_active_lanes", 32.0)
                                                           / max(1, E))
        if cnt.get("dram_bytes") is not None:
            measured["dram_util"] = cnt["dram_bytes"] / t_s / hbm_peak
    prefix_util = bytes_prefix / t_s / hbm_peak
    mem_util = max(prefix_util, measured.get("dram_util", 0.0))
    issue_util = measured.get("issue_util", ops / t_s / fp32_peak)
    bound = "issue" if issue_util >= mem_util else "hbm"
    if bound == "issue":
        head = {"achieved": ops / t_s / 1e9, "peak": fp32_peak / 1e9, "unit": "Ginstr/s (FP32 lanes)",
                "frac": ops / t_s / fp32_peak,
                "work_def": "SURVEY 8d: 16 FP32-pipe instructions per evaluated pair E + 8 per committed pair C",
                "algorithmic_work": ops}
    else:
        head = {"achieved": bytes_alg / t_s / 1e9, "peak": hbm_peak / 1e9, "unit": "GB/s",
                "frac": bytes_alg / t_s / hbm_peak,
                "work_def": "SURVEY 8d: 44 B per tile instance + 32 B per output pixel", "algorithmic_work": bytes_alg}
    res["roofline"] = dict(
        {"bound": bound, "bound_basis": ("measured: issue_util (ncu warp instructions / (148 SMs x 4 x clock x t)) "
                                         f"{issue_util:.3f} vs memory util (max of consumed-prefix bytes and ncu DRAM "
                                         f"bytes / (HBM peak x t)) {mem_util:.3f}"),
         "kernel": kname, "t_ms": t_s * 1e3},
        **head,
        traffic=measured.get("dram_bytes", traffic), measured=measured,
        t_roof_ms=t_roof * 1e3, t_roof_frac=t_roof / t_s,
        t_roof_def=("max(16E+8C / FP32 peak, E / MUFU peak, consumed-prefix bytes / HBM peak): SURVEY 8d's terms, "
                    "the HBM term over the bytes blending must read"),
        t_roof_survey_ms=t_roof_survey * 1e3, t_roof_survey_frac=t_roof_survey / t_s,
        t_roof_survey_def="SURVEY 8d as written: max(16E+8C / FP32 peak, E / MUFU peak, (44K+32P) / HBM peak)",
        api_kernel_view=api_view, peak_source=hbm_src,
        hbm_view={"achieved": bytes_alg / t_s / 1e9, "peak": hbm_peak / 1e9, "unit": "GB/s",
                  "frac": bytes_alg / t_s / hbm_peak, "algorithmic_bytes": bytes_alg},
        consumed_prefix_view={
            "bytes": bytes_prefix, "frac": prefix_util,
            "def": "44 B per entry of each tile's longest consumed list prefix + 32 B per pixel: what tile-serial "
                   "blending must read; K*44 exceeds it when list tails lie past every pixel's stop"},
        issue_view={"achieved_ginstr_s": ops / t_s / 1e9, "peak_ginstr_s": fp32_peak / 1e9,
                    "frac": (ops / t_s) / fp32_peak, "ops": ops,
                    "def": "FP32-pipe instructions 16E+8C (SURVEY 8d), peak 148 SMs x 128 lanes x sm_max_mhz"},
        mufu_view={"frac": (E / t_s) / mufu_peak})

    # C3: the imbalance sweep on the C2 geometry — render time of
    # the pixel-wise baseline vs the balanced kernels at every point, the
    # north-star ratio FG / Naive on the most imbalanced scene, and the
    # per-frame selector's choice and regret
    if not args.no_c3:
        res["c3_sweep"] = c3_sweep(api, N, torch, W, H, pw, ph, n, cams[0].focal[0], mode, dev)

    # e2e: the same metric through the C-ABI with HOST buffers, host<->device
    # copies inside the timed region.  Batch mode (the timed steps' shape):
    # each step is one bs_render_views_host call — the scene uploaded once
    # from pinned host memory, the step's 64 views rendered round-robin over
    # min(--streams, 4) contexts (async frame bodies; C1 with 8 host-buffer
    # contexts measured 10.2k vs 11.3k views/s with 4), every view's six output planes
    # downloaded into its own pinned host buffers; --batch 0: one
    # bs_render_frame_host_async call (scene upload + frame + download) per
    # view.  Wall clock from the first enqueue to bs_context_sync on every
    # context.
    nctx = max(1, min(args.streams, 4))
    ctxs = []
    for _ in range(nctx):
        cx = C.c_void_p()
        N.call("bs_context_create", C.byref(cx), int(mode))
        N.call("bs_context_set_async", cx, 1)
        if nctx > 1:
            N.call("bs_context_set_fine_occupancy", cx, args.fine_ctas)
        ctxs.append(cx)
    host_g3d = torch.from_numpy(np.ascontiguousarray(g3d).view(np.uint8).reshape(-1).copy()).pin_memory()
    P3 = P * 3
    bgc = (C.c_float * 3)(0.0, 0.0, 0.0)
    vv = -1 if args.variant == "auto" else int(vsel)

    def e2e_sync():
        tot = 0
        for cx in ctxs:
            r = C.c_int64(0)
            N.call("bs_context_sync", cx, C.byref(r))
            tot += r.value
        return tot

    batch = max(0, args.batch)
    if batch:
        # one pinned output set per view of the batch (every view's result lands on the host)
        outs = [[torch.empty(P3, dtype=torch.float32).pin_memory()] +
                [torch.empty(P, dtype=torch.float32).pin_memory() for _ in range(3)] +
                [torch.empty(P, dtype=torch.int32).pin_memory() for _ in range(2)] for _ in range(batch)]
        out_ptrs = (C.c_void_p * (6 * batch))(*[o.data_ptr() for v in outs for o in v])
        ctx_arr = (C.c_void_p * nctx)(*[cx.value for cx in ctxs])
        cam_arr = (N.Camera * N_VIEWS)(*cams)
        ids = (C.c_int32 * batch)(*[k % N_VIEWS for k in range(batch)])

        def e2e_step(_k):
            N.call("bs_render_views_host", ctx_arr, nctx, host_g3d.data_ptr(), n, cam_arr, ids, batch, pw, ph, vv,
                   bgc, out_ptrs)
        per_step, warm, ne = batch, 2, max(3, min(args.steps, 10))
        h2d, path = int(n * 56), ("bs_render_views_host (C-ABI; the scene uploaded once per step from pinned host "
                                  "memory, the step's views round-robin over the contexts, each view's six planes "
                                  "downloaded into its own pinned host buffers; wall clock to bs_context_sync)")
    else:
        rings = [[[torch.empty(P3, dtype=torch.float32).pin_memory()] +
                  [torch.empty(P, dtype=torch.float32).pin_memory() for _ in range(3)] +
                  [torch.empty(P, dtype=torch.int32).pin_memory() for _ in range(2)] for _ in range(3)]
                 for _ in range(nctx)]

        def e2e_step(k):
            c_, j = k % nctx, k // nctx
            N.call("bs_render_frame_host_async", ctxs[c_], host_g3d.data_ptr(), n, C.byref(cams[k % N_VIEWS]), pw,
                   ph, vv, bgc, *[o.data_ptr() for o in rings[c_][j % 3]])
        per_step, warm, ne = 1, 4 * nctx, max(3, min(args.steps, 100))
        h2d, path = int(n * 56), ("bs_render_frame_host_async (C-ABI; pinned host buffers; per context upload / "
                                  "frame / download on three streams, 3 frames in flight; frames round-robin over "
                                  "the contexts; wall clock to bs_context_sync)")
    for k in range(warm):
        e2e_step(k)
    r0 = e2e_sync()
    t0 = time.perf_counter()
    for k in range(ne):
        e2e_step(k)
    r1 = e2e_sync()
    e2e_s = (time.perf_counter() - t0) / ne
    for cx in ctxs:
        N.call("bs_context_destroy", cx)
    res["e2e"] = {"value": per_step / e2e_s, "unit": "views/s", "h2d_bytes_per_step": h2d,
                  "d2h_bytes_per_step": int(P * 32) * per_step, "views_per_step": per_step,
                  "ms_per_step": e2e_s * 1e3, "steps": ne, "reruns": int(r1 - r0), "contexts": nctx, "path": path}

    if world == 1 and not args.no_cpu_baseline:
        g2d = api.splats_to_g2d(s)
        pl = b.point_list.cpu().numpy().view(np.uint32)
        ranges = b.tile_ranges.cpu().numpy().view(np.uint32)
        O, R, kind = cpu_libs()
        ocam = O.Camera.from_buffer_copy(bytes(cam_id))
        tcpu, parts, desc = cpu_sample_estimate(O, R, g3d.view(O.G3D_DTYPE), ocam, g2d.view(O.G2D_DTYPE), pl, ranges,
                                                W, H, pw, ph, args.cpu_budget, variant=3)
        res["cpu_baseline"] = {"value": 1.0 / tcpu, "unit": "views/s", "cores": 1, "kind": kind, "sample": desc,
                               "stage_s": parts, "host_cpu": os.cpu_count()}
    return res


if __name__ == "__main__":
    main()
