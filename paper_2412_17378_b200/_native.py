"""ctypes binding of the C-ABI in include/splatsim_b200.h.

Loads the in-tree ``lib/libsplatsim_b200.so`` (built by ``__graft_entry__.build()``
/ ``make -C paper_2412_17378_b200``).  There is no fallback: if the library is
missing, importing the product API raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libsplatsim_b200.so")

# ---- structs (must match include/splatsim_b200.h) ----


class Camera(C.Structure):
    _fields_ = [("view", C.c_float * 16), ("focal", C.c_float * 2), ("width", C.c_int32), ("height", C.c_int32)]


class Splats(C.Structure):
    _fields_ = [("xyab", C.c_void_p), ("cop", C.c_void_p), ("rgbr", C.c_void_p)]


class FrameOut(C.Structure):
    _fields_ = [("color", C.c_void_p), ("alpha", C.c_void_p), ("depth", C.c_void_p), ("final_t", C.c_void_p),
                ("contrib", C.c_void_p), ("term", C.c_void_p)]


class FrameGradIn(C.Structure):
    _fields_ = [("dl_dcolor", C.c_void_p), ("dl_dalpha", C.c_void_p), ("dl_ddepth", C.c_void_p)]


class SplatGrads(C.Structure):
    _fields_ = [("xyab", C.c_void_p), ("cop", C.c_void_p), ("rgbr", C.c_void_p)]


class TileHistogram(C.Structure):
    _fields_ = [("min", C.c_uint32), ("max", C.c_uint32), ("p50", C.c_uint32), ("p99", C.c_uint32),
                ("mean", C.c_double), ("total", C.c_uint64), ("tiles", C.c_int32), ("nonempty", C.c_int32)]


class TrainingParams(C.Structure):
    _fields_ = [("total_iters", C.c_int32), ("keyframes", C.c_int32), ("width", C.c_int32), ("height", C.c_int32),
                ("patch_width", C.c_int32), ("patch_height", C.c_int32), ("focal", C.c_float),
                ("n_gaussians", C.c_int32), ("seed", C.c_uint64),
                ("background_fraction_start", C.c_double), ("background_fraction_end", C.c_double),
                ("cluster_sigma_start", C.c_double), ("cluster_sigma_end", C.c_double),
                ("opacity_scale_start", C.c_double), ("opacity_scale_end", C.c_double)]


class FrameInfo(C.Structure):
    _fields_ = [("variant", C.c_int32), ("n_visible", C.c_int32), ("k", C.c_int64), ("stats", TileHistogram),
                ("evaluated", C.c_uint64), ("committed", C.c_uint64)]


G3D_DTYPE = np.dtype([("mean", "<f4", 3), ("scale", "<f4", 3), ("rot", "<f4", 4), ("opacity", "<f4"),
                      ("color", "<f4", 3)])
G2D_DTYPE = np.dtype([("x", "<f4"), ("y", "<f4"), ("conic_a", "<f4"), ("conic_b", "<f4"), ("conic_c", "<f4"),
                      ("opacity", "<f4"), ("color", "<f4", 3), ("depth", "<f4"), ("radius", "<f4")])
assert G3D_DTYPE.itemsize == 56 and G2D_DTYPE.itemsize == 44
TILE_HIST_DTYPE_BYTES = C.sizeof(TileHistogram)

VARIANTS = ("Naive", "DynamicBlocks", "GaussianWise", "FineGrainedCombined", "SharedMemOpt")
ALPHA_EXACT, ALPHA_FAST = 0, 1

# C-ABI exports: name -> (restype, argtypes)
_vp, _i32, _i64, _u64, _sz, _f32p = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_size_t, C.POINTER(C.c_float)
SIGNATURES = {
    "bs_abi_version": (C.c_int, []),
    "bs_status_string": (C.c_char_p, [C.c_int]),
    "bs_device_sm_count": (C.c_int, [C.POINTER(C.c_int32)]),
    "bs_variant_name": (C.c_char_p, [C.c_int]),
    "bs_variant_from_name": (C.c_int, [C.c_char_p]),
    "bs_preprocess_workspace_bytes": (_sz, [_i64]),
    "bs_preprocess": (C.c_int, [_vp, _i64, C.POINTER(Camera), Splats, _vp, _vp, _sz, _vp]),
    "bs_splats_from_g2d": (C.c_int, [_vp, _i64, Splats, _vp]),
    "bs_splats_to_g2d": (C.c_int, [Splats, _i64, _vp, _vp]),
    "bs_bin_workspace_bytes": (_sz, [_i64, _i32, _i32, _i32, _i32, _i64]),
    "bs_bin_count": (C.c_int, [Splats, _i64, _vp, _i32, _i32, _i32, _i32, _vp, _vp, _sz, _vp]),
    "bs_preprocess_bin_count": (C.c_int, [_vp, _i64, C.POINTER(Camera), _vp, Splats, _vp, _i32, _i32, _i32, _i32, _vp,
                                          _vp, _sz, _vp]),
    "bs_bin_sort": (C.c_int, [Splats, _i64, _vp, _i32, _i32, _i32, _i32, _i64, _vp, _vp, _vp, _sz, _vp]),
    "bs_tile_stats_workspace_bytes": (_sz, [_i32]),
    "bs_tile_stats": (C.c_int, [_vp, _i32, _vp, _vp, _vp, _vp, _sz, _vp]),
    "bs_tile_order": (C.c_int, [_vp, _i32, _vp, _vp, _vp]),
    "bs_render_workspace_bytes": (_sz, [_i32, _i32]),
    "bs_render_forward": (C.c_int, [C.c_int, C.c_int, Splats, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _f32p,
                                    FrameOut, _vp, _sz, _vp]),
    "bs_frame_work": (C.c_int, [_vp, _vp, _vp, _i32, _i32, _i32, _i32, _vp, _vp]),
    "bs_render_set_fine_occupancy": (C.c_int, [_i32]),
    "bs_render_forward_ctx": (C.c_int, [C.c_int, _vp, C.c_int, Splats, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _f32p,
                                        FrameOut, _i32, _i32, _vp, _sz, _vp]),
    "bs_select_variant": (C.c_int, [C.POINTER(TileHistogram), _i32, _i32, _i32, _i32, _i32]),
    "bs_test_expf": (C.c_int, [_vp, _vp, _i64, C.c_int, _vp]),
    "bs_test_expf_range": (C.c_int, [C.c_uint32, _i64, _vp, C.c_int, _vp]),
    "bs_context_create": (C.c_int, [C.POINTER(C.c_void_p), C.c_int]),
    "bs_context_destroy": (C.c_int, [_vp]),
    "bs_context_stream": (_vp, [_vp]),
    "bs_render_frame_host": (C.c_int, [_vp, _vp, _i64, C.POINTER(Camera), _i32, _i32, _i32, _f32p, _vp, _vp, _vp,
                                       _vp, _vp, _vp, _vp]),
    "bs_render_frame_host_async": (C.c_int, [_vp, _vp, _i64, C.POINTER(Camera), _i32, _i32, _i32, _f32p, _vp, _vp,
                                             _vp, _vp, _vp, _vp]),
    "bs_render_frame_device": (C.c_int, [_vp, _vp, _i64, C.POINTER(Camera), _i32, _i32, _i32, _f32p, FrameOut,
                                         _vp]),
    "bs_context_set_stream": (C.c_int, [_vp, _vp]),
    "bs_context_frame": (C.c_int, [_vp, C.POINTER(FrameOut)]),
    "bs_publish_i64": (C.c_int, [_vp, _vp, _vp]),
    "bs_super_aux_bytes": (_sz, [_i32, _i32, _i32, _i32]),
    "bs_preprocess_bin_count_super": (C.c_int, [_vp, _i64, C.POINTER(Camera), _vp, Splats, _vp, _i32, _i32, _i32,
                                                _i32, _vp, _vp, _sz, _vp, _vp, _sz, _vp]),
    "bs_render_backward": (C.c_int, [C.c_int, Splats, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _f32p, FrameOut,
                                     FrameGradIn, SplatGrads, C.c_int, _vp, _sz, _vp]),
    "bs_context_render_backward": (C.c_int, [_vp, FrameGradIn, SplatGrads]),
    "bs_render_forward_super": (C.c_int, [C.c_int, _vp, C.c_int, Splats, _vp, _vp, _vp, _i32, _i32, _i32, _i32,
                                          _f32p, FrameOut, _vp, _sz, _vp]),
    "bs_super_tile_ranges": (C.c_int, [_vp, _i32, _i32, _i32, _i32, _vp, _vp]),
    "bs_super_tile_lengths": (C.c_int, [_vp, _sz, _i32, _i32, _i32, _i32, _vp, _vp]),
    "bs_tile_order_select": (C.c_int, [_vp, _i32, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _vp, _vp]),
    "bs_context_list_mode": (C.c_int, [_vp, C.POINTER(C.c_int32)]),
    "bs_render_views_host": (C.c_int, [_vp, _i32, _vp, _i64, _vp, _vp, _i32, _i32, _i32, _i32, _f32p, _vp]),
    "bs_render_views": (C.c_int, [C.POINTER(C.c_void_p), _i32, _vp, _i64, C.POINTER(Camera), C.POINTER(C.c_int32),
                                  _i32, _i32, _i32, _i32, _f32p, C.POINTER(C.c_void_p), _sz]),
    "bs_context_set_async": (C.c_int, [_vp, _i32]),
    "bs_context_sync": (C.c_int, [_vp, C.POINTER(C.c_int64)]),
    "bs_context_capacity": (C.c_int, [_vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "bs_context_drop_pending": (C.c_int, [_vp]),
    "bs_context_set_graphs": (C.c_int, [_vp, _i32]),
    "bs_context_set_fine_occupancy": (C.c_int, [_vp, _i32]),
    "bs_context_graph_launches": (C.c_int, [_vp, C.POINTER(C.c_int64)]),
    "bs_preprocess_devcam": (C.c_int, [_vp, _i64, _vp, Splats, _vp, _vp, _sz, _vp]),
    "bs_bin_sort_async": (C.c_int, [Splats, _i64, _vp, _i32, _i32, _i32, _i32, _i64, _vp, _vp, _vp, _sz, _vp]),
    "bs_bin_async_supported": (C.c_int, [_i32, _i32, _i32, _i32]),
    "bs_context_last_info": (C.c_int, [_vp, C.POINTER(FrameInfo)]),
    "bs_context_enable_timing": (C.c_int, [_vp, _i32]),
    "bs_context_stage_ms": (C.c_int, [_vp, _f32p, _i32]),
    "bs_select_variant_device": (C.c_int, [_vp, _i32, _i32, _i32, _i32, _i32, _vp, _vp]),
    "bs_render_forward_auto": (C.c_int, [_vp, C.c_int, Splats, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _f32p,
                                         FrameOut, _vp, _sz, _vp]),
    "bs_host_run_training": (C.c_int, [C.POINTER(TrainingParams), _i32, C.c_char_p, _sz, C.POINTER(C.c_size_t)]),
    "bs_kernel_launches": (_u64, []),
    "bs_host_gen_clustered_scene": (C.c_int, [_i32, _i32, _u64, C.c_double, C.c_double, C.POINTER(Camera), _vp]),
}


class BsError(RuntimeError):
    def __init__(self, fn: str, status: int, msg: str):
        super().__init__(f"{fn} failed: {msg} (status {status})")
        self.status = status


_lib = None


def lib() -> C.CDLL:
    """Load and type the native library (raises if absent — no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"native library missing: {LIB_PATH} (run __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(fn: str, status: int) -> None:
    if status != 0:
        raise BsError(fn, status, lib().bs_status_string(status).decode())


def call(fn: str, *args) -> int:
    st = getattr(lib(), fn)(*args)
    check(fn, st)
    return st


def make_camera(view=None, focal=(100.0, 100.0), width=0, height=0) -> Camera:
    cam = Camera()
    v = np.eye(4, dtype=np.float32) if view is None else np.asarray(view, dtype=np.float32).reshape(4, 4)
    for i, x in enumerate(v.reshape(-1)):
        cam.view[i] = float(x)
    cam.focal[0], cam.focal[1] = float(focal[0]), float(focal[1])
    cam.width, cam.height = int(width), int(height)
    return cam


def camera_to_numpy(cam: Camera) -> np.ndarray:
    return np.frombuffer(bytes(cam), dtype=np.uint8).copy()
