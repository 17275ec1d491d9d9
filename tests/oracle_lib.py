"""ctypes access to the CPU oracle (oracle/_build/liboracle.so).

TEST INFRASTRUCTURE: the oracle is the parity checker, never the product.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
ORACLE_LIB = os.path.join(ORACLE_DIR, "_build", "liboracle.so")

G3D_DTYPE = np.dtype([("mean", "<f4", 3), ("scale", "<f4", 3), ("rot", "<f4", 4), ("opacity", "<f4"),
                      ("color", "<f4", 3)])
G2D_DTYPE = np.dtype([("x", "<f4"), ("y", "<f4"), ("conic_a", "<f4"), ("conic_b", "<f4"), ("conic_c", "<f4"),
                      ("opacity", "<f4"), ("color", "<f4", 3), ("depth", "<f4"), ("radius", "<f4")])


class Camera(C.Structure):
    _fields_ = [("view", C.c_float * 16), ("focal", C.c_float * 2), ("width", C.c_int32), ("height", C.c_int32)]


def make_camera(view=None, focal=(100.0, 100.0), width=0, height=0) -> Camera:
    cam = Camera()
    v = np.eye(4, dtype=np.float32) if view is None else np.asarray(view, dtype=np.float32).reshape(4, 4)
    for i, x in enumerate(v.reshape(-1)):
        cam.view[i] = float(x)
    cam.focal[0], cam.focal[1] = float(focal[0]), float(focal[1])
    cam.width, cam.height = int(width), int(height)
    return cam


_lib = None


def build() -> None:
    subprocess.run(["make", "-s", "-C", ORACLE_DIR], check=True)


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_LIB):
            build()
        L = C.CDLL(ORACLE_LIB)
        vp, i64, i32, f32, f64 = C.c_void_p, C.c_int64, C.c_int32, C.c_float, C.c_double
        L.orc_gen_clustered_scene.argtypes = [C.c_int, C.c_int, C.c_uint64, f64, f64, C.POINTER(Camera), vp]
        L.orc_covariance_of.argtypes = [vp, vp]
        L.orc_project_covariance.argtypes = [vp, vp, vp, vp]
        L.orc_project_gaussian.argtypes = [vp, C.POINTER(Camera), vp]
        L.orc_project_all.argtypes = [vp, i64, C.POINTER(Camera), vp]
        L.orc_project_all.restype = i64
        L.orc_bin_tiles.argtypes = [vp, i64, C.c_int, C.c_int, C.c_int, C.c_int, vp, i64, vp]
        L.orc_bin_tiles.restype = i64
        L.orc_tile_load_histogram.argtypes = [vp, C.c_int, C.c_int, vp, vp, vp, vp, vp, vp]
        L.orc_eval_alpha.argtypes = [vp, f32, f32, vp, vp]
        L.orc_blend_pixel.argtypes = [C.c_int, vp, vp, vp, C.c_int, vp, vp, vp, vp, vp, vp, vp]
        L.orc_termination_index.argtypes = [vp, C.c_int]
        L.orc_warp_prefix_product_f32.argtypes = [vp, f32, vp, vp]
        L.orc_warp_prefix_product_f64.argtypes = [vp, f64, vp, vp]
        L.orc_render.argtypes = [C.c_int, vp, vp, i64, vp, i64, C.c_int, C.c_int, C.c_int, C.c_int, vp, C.c_int,
                                 C.c_int, vp, C.c_int, vp, vp, vp, vp, vp, vp]
        L.orc_warp_steps_pixelwise.argtypes = [vp, C.c_int, i64]
        L.orc_warp_steps_pixelwise.restype = i64
        L.orc_warp_steps_gaussianwise.argtypes = [i64, i64]
        L.orc_warp_steps_gaussianwise.restype = i64
        L.orc_fnv1a64.argtypes = [vp, C.c_size_t, C.c_uint64]
        L.orc_fnv1a64.restype = C.c_uint64
        L.orc_libm_expf.argtypes = [f32]
        L.orc_libm_expf.restype = f32
        L.orc_expf_exhaustive_check.argtypes = [f32, f32, vp, C.c_int]
        L.orc_expf_exhaustive_check.restype = i64
        L.orc_expf_compare_batch.argtypes = [vp, vp, i64]
        L.orc_expf_compare_batch.restype = i64
        L.orc_expf_compare_range.argtypes = [C.c_uint32, i64, vp]
        L.orc_expf_compare_range.restype = i64
        L.orc_render_backward.argtypes = [vp, vp, i64, vp, i64, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp, vp, vp,
                                          vp]
        _lib = L
    return _lib


def p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data


def gen_clustered_scene(n, cam, n_clusters=4, seed=42, sigma=0.035, bgfrac=0.12) -> np.ndarray:
    out = np.zeros(int(n), dtype=G3D_DTYPE)
    rc = lib().orc_gen_clustered_scene(int(n), int(n_clusters), int(seed), float(sigma), float(bgfrac), C.byref(cam),
                                       p(out) if n else None)
    assert rc == 0
    return out


def project_all(g3d: np.ndarray, cam) -> np.ndarray:
    out = np.zeros(max(len(g3d), 1), dtype=G2D_DTYPE)
    m = lib().orc_project_all(p(g3d), len(g3d), C.byref(cam), p(out))
    return out[:m].copy()


def bin_tiles(g2d: np.ndarray, W, H, pw, ph):
    cols, rows = (W + pw - 1) // pw, (H + ph - 1) // ph
    ranges = np.zeros(2 * cols * rows, dtype=np.uint32)
    K = lib().orc_bin_tiles(p(g2d), len(g2d), W, H, pw, ph, None, 0, p(ranges))
    pl = np.zeros(max(K, 1), dtype=np.uint32)
    K2 = lib().orc_bin_tiles(p(g2d), len(g2d), W, H, pw, ph, p(pl), K, p(ranges))
    assert K == K2
    return pl[:K].copy(), ranges


def tile_load_histogram(ranges: np.ndarray, cols: int, rows: int) -> dict:
    counts = np.zeros(max(cols * rows, 1), dtype=np.uint32)
    mn, mx, p50, p99 = (C.c_uint32() for _ in range(4))
    mean = C.c_double()
    lib().orc_tile_load_histogram(p(ranges), cols, rows, p(counts), C.byref(mn), C.byref(mx), C.byref(mean),
                                  C.byref(p50), C.byref(p99))
    return {"counts": counts[: cols * rows], "min": mn.value, "max": mx.value, "mean": mean.value, "p50": p50.value,
            "p99": p99.value}


def render(variant: int, pl, ranges, g2d, W, H, pw, ph, bg=(0, 0, 0), lazy=True, threads=0, tiles=None) -> dict:
    P = W * H
    out = {"color": np.zeros(3 * P, np.float32), "alpha": np.zeros(P, np.float32), "depth": np.zeros(P, np.float32),
           "final_t": np.zeros(P, np.float32), "contrib": np.zeros(P, np.int32), "term": np.zeros(P, np.int32)}
    bgc = np.asarray(bg, dtype=np.float32)
    pl = np.ascontiguousarray(pl, dtype=np.uint32)
    if len(pl) == 0:
        pl = np.zeros(1, np.uint32)
    t = None if tiles is None else np.ascontiguousarray(tiles, dtype=np.int32)
    rc = lib().orc_render(int(variant), p(ranges), p(pl), len(pl), p(g2d) if len(g2d) else None, len(g2d), W, H, pw,
                          ph, p(bgc), int(lazy), int(threads), p(t), 0 if t is None else len(t), p(out["color"]),
                          p(out["alpha"]), p(out["depth"]), p(out["final_t"]), p(out["contrib"]), p(out["term"]))
    assert rc == 0, rc
    return out


def blend_pixel(alphas, colors=None, depths=None, bg=(0, 0, 0), gaussianwise=False) -> dict:
    a = np.ascontiguousarray(alphas, dtype=np.float32)
    n = len(a)
    col = None if colors is None else np.ascontiguousarray(colors, dtype=np.float32).reshape(-1)
    dep = None if depths is None else np.ascontiguousarray(depths, dtype=np.float32)
    bgc = np.asarray(bg, dtype=np.float32)
    oc = np.zeros(3, np.float32)
    oa, od, ot = C.c_float(), C.c_float(), C.c_float()
    cc, tt = C.c_int32(), C.c_int32()
    lib().orc_blend_pixel(int(gaussianwise), p(a) if n else None, p(col), p(dep), n, p(bgc), p(oc), C.byref(oa),
                          C.byref(od), C.byref(ot), C.byref(cc), C.byref(tt))
    return {"color": oc, "alpha": oa.value, "depth": od.value, "final_t": ot.value, "contrib": cc.value,
            "term": tt.value}


def fnv1a64(arr: np.ndarray, h: int = 0xCBF29CE484222325) -> int:
    b = np.ascontiguousarray(arr)
    return int(lib().orc_fnv1a64(p(b), b.nbytes, h))


GRAD_FIELDS = ("x", "y", "conic_a", "conic_b", "conic_c", "opacity", "r", "g", "b", "depth")


def render_backward(pl, ranges, g2d, W, H, pw, ph, bg, dl_dcolor, dl_dalpha, dl_ddepth) -> np.ndarray:
    """Per-splat gradients (n x 10, GRAD_FIELDS order, float64) of render_reference's outputs."""
    n = len(g2d)
    out = np.zeros((max(n, 1), 10), np.float64)
    pl = np.ascontiguousarray(pl, dtype=np.uint32)
    if len(pl) == 0:
        pl = np.zeros(1, np.uint32)
    bgc = np.asarray(bg, dtype=np.float32)
    dc = np.ascontiguousarray(dl_dcolor, dtype=np.float32)
    da = np.ascontiguousarray(dl_dalpha, dtype=np.float32)
    dd = np.ascontiguousarray(dl_ddepth, dtype=np.float32)
    rc = lib().orc_render_backward(p(np.ascontiguousarray(ranges, dtype=np.uint32)), p(pl), len(pl),
                                   p(g2d) if n else None, n, W, H, pw, ph, p(bgc), p(dc), p(da), p(dd), p(out))
    assert rc == 0, rc
    return out[:n]
