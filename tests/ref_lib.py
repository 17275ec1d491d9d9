"""ctypes access to the REFERENCE ITSELF (oracle/_ref/libsplatsim_ref.so):
/root/reference/proj/core's unmodified sources compiled against the in-repo
Eigen-subset shim (oracle/Makefile, target ``ref``; oracle/ref_capi.cpp).

TEST INFRASTRUCTURE: it pins the oracle restatement (oracle/) and the golden
fixtures to the reference's own code.  The library is built here (where
/root/reference exists) and travels to the GPU box as a built file; when it is
neither built nor buildable, ``available()`` is False and its tests skip.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

import oracle_lib as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libsplatsim_ref.so")
REF_SRC = "/root/reference/proj/core/src"

_lib = None


def available() -> bool:
    if os.path.exists(REF_LIB):
        return True
    if os.path.isdir(REF_SRC):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)
        return os.path.exists(REF_LIB)
    return False


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        assert available(), "oracle/_ref not built and /root/reference absent"
        L = C.CDLL(REF_LIB)
        vp, i64, f32, f64, cp = C.c_void_p, C.c_int64, C.c_float, C.c_double, C.c_char_p
        I = C.c_int
        L.ref_gen_clustered_scene.argtypes = [I, I, C.c_uint64, f64, f64, C.POINTER(O.Camera), vp]
        L.ref_covariance_of.argtypes = [vp, vp]
        L.ref_project_covariance.argtypes = [vp, vp, vp, vp]
        L.ref_project_gaussian.argtypes = [vp, C.POINTER(O.Camera), vp]
        L.ref_project_all.argtypes = [vp, i64, C.POINTER(O.Camera), vp, I]
        L.ref_project_all.restype = i64
        L.ref_bin_tiles.argtypes = [vp, i64, I, I, I, I, vp, i64, vp]
        L.ref_bin_tiles.restype = i64
        L.ref_tile_load_histogram.argtypes = [vp, I, I, vp, vp, vp, vp, vp, vp]
        L.ref_binning_csv.argtypes = [vp, I, I, cp, vp, C.c_size_t]
        L.ref_eval_alpha.argtypes = [vp, f32, f32, vp, vp]
        L.ref_blend_pixel.argtypes = [vp, vp, vp, I, vp, vp, vp, vp, vp, vp, vp]
        L.ref_termination_index.argtypes = [vp, I]
        L.ref_warp_prefix_product_f32.argtypes = [vp, f32, vp, vp]
        L.ref_run_kernel.argtypes = [I, vp, vp, i64, vp, i64, I, I, I, I, vp, I, vp, vp, vp, vp, vp, vp, vp,
                                     C.c_size_t]
        L.ref_make_task_specs.argtypes = [I, I, I, I, I, vp, vp, vp, i64]
        L.ref_make_task_specs.restype = i64
        L.ref_trace_csv.argtypes = [I, vp, vp, I, I, cp, vp, C.c_size_t]
        L.ref_warp_steps_pixelwise.argtypes = [vp, I, i64]
        L.ref_warp_steps_pixelwise.restype = i64
        L.ref_warp_steps_gaussianwise.argtypes = [i64, i64]
        L.ref_warp_steps_gaussianwise.restype = i64
        L.ref_write_ppm.argtypes = [I, I, vp, cp]
        L.ref_write_float_grid.argtypes = [vp, i64, I, I, cp]
        L.ref_render_digest_csv.argtypes = [I, I, vp, vp, vp, vp, vp, vp, cp, vp, C.c_size_t]
        L.ref_compare_outputs.argtypes = [I, I, vp, vp, I, I, vp, vp, vp, vp, vp]
        L.ref_scene_roundtrip.argtypes = [cp, vp, C.c_size_t]
        L.ref_serialize_scene.argtypes = [C.POINTER(O.Camera), I, I, vp, C.c_uint64, vp, i64, vp, C.c_size_t]
        L.ref_fnv1a64.argtypes = [vp, C.c_size_t, C.c_uint64]
        L.ref_fnv1a64.restype = C.c_uint64
        _lib = L
    return _lib


p = O.p


def _string(fn, *args) -> tuple[int, str]:
    """Calls a string-returning entry point twice: size, then content."""
    n = fn(*args, None, 0)
    buf = C.create_string_buffer(abs(n) + 1)
    rc = fn(*args, buf, len(buf))
    return rc, buf.value.decode()


def gen_clustered_scene(n, cam, n_clusters=4, seed=42, sigma=0.035, bgfrac=0.12) -> np.ndarray:
    out = np.zeros(int(n), dtype=O.G3D_DTYPE)
    rc = lib().ref_gen_clustered_scene(int(n), int(n_clusters), int(seed), float(sigma), float(bgfrac),
                                       C.byref(cam), p(out) if n else None)
    assert rc == 0
    return out


def project_all(g3d: np.ndarray, cam, threads: int = 1) -> np.ndarray:
    out = np.zeros(max(len(g3d), 1), dtype=O.G2D_DTYPE)
    m = lib().ref_project_all(p(g3d), len(g3d), C.byref(cam), p(out), int(threads))
    return out[:m].copy()


def bin_tiles(g2d: np.ndarray, W, H, pw, ph):
    cols, rows = (W + pw - 1) // pw, (H + ph - 1) // ph
    ranges = np.zeros(2 * cols * rows, dtype=np.uint32)
    K = lib().ref_bin_tiles(p(g2d), len(g2d), W, H, pw, ph, None, 0, p(ranges))
    pl = np.zeros(max(K, 1), dtype=np.uint32)
    lib().ref_bin_tiles(p(g2d), len(g2d), W, H, pw, ph, p(pl), K, p(ranges))
    return pl[:K].copy(), ranges


def tile_load_histogram(ranges, cols, rows) -> dict:
    counts = np.zeros(max(cols * rows, 1), dtype=np.uint32)
    mn, mx, p50, p99 = (C.c_uint32() for _ in range(4))
    mean = C.c_double()
    lib().ref_tile_load_histogram(p(ranges), cols, rows, p(counts), C.byref(mn), C.byref(mx), C.byref(mean),
                                  C.byref(p50), C.byref(p99))
    return {"counts": counts[: cols * rows], "min": mn.value, "max": mx.value, "mean": mean.value, "p50": p50.value,
            "p99": p99.value}


def run_kernel(variant, pl, ranges, g2d, W, H, pw, ph, bg=(0, 0, 0), threads=1, trace=False):
    P = W * H
    out = {"color": np.zeros(3 * P, np.float32), "alpha": np.zeros(P, np.float32), "depth": np.zeros(P, np.float32),
           "final_t": np.zeros(P, np.float32), "contrib": np.zeros(P, np.int32), "term": np.zeros(P, np.int32)}
    bgc = np.asarray(bg, dtype=np.float32)
    pl = np.ascontiguousarray(pl, dtype=np.uint32)
    if len(pl) == 0:
        pl = np.zeros(1, np.uint32)
    tbuf = C.create_string_buffer(64 << 20) if trace else None
    rc = lib().ref_run_kernel(int(variant), p(ranges), p(pl), len(pl), p(g2d) if len(g2d) else None, len(g2d), W, H,
                              pw, ph, p(bgc), int(threads), p(out["color"]), p(out["alpha"]), p(out["depth"]),
                              p(out["final_t"]), p(out["contrib"]), p(out["term"]), tbuf, len(tbuf) if trace else 0)
    assert rc == 0, rc
    if trace:
        out["trace_csv"] = tbuf.value.decode()
    return out


def blend_pixel(alphas, colors=None, depths=None, bg=(0, 0, 0)) -> dict:
    a = np.ascontiguousarray(alphas, dtype=np.float32)
    n = len(a)
    col = None if colors is None else np.ascontiguousarray(colors, dtype=np.float32).reshape(-1)
    dep = None if depths is None else np.ascontiguousarray(depths, dtype=np.float32)
    bgc = np.asarray(bg, dtype=np.float32)
    oc = np.zeros(3, np.float32)
    oa, od, ot = C.c_float(), C.c_float(), C.c_float()
    cc, tt = C.c_int32(), C.c_int32()
    lib().ref_blend_pixel(p(a) if n else None, p(col), p(dep), n, p(bgc), p(oc), C.byref(oa), C.byref(od),
                          C.byref(ot), C.byref(cc), C.byref(tt))
    return {"color": oc, "alpha": oa.value, "depth": od.value, "final_t": ot.value, "contrib": cc.value,
            "term": tt.value}


def trace_csv(variant, list_len: np.ndarray, consumed: np.ndarray, comment="ref") -> str:
    ll = np.ascontiguousarray(list_len, dtype=np.int32)
    cons = np.ascontiguousarray(consumed, dtype=np.int32)
    T, cap = cons.shape
    return _string(lib().ref_trace_csv, int(variant), p(ll), p(cons), T, cap, comment.encode())[1]


def make_task_specs(variant, W, H, pw, ph):
    n = lib().ref_make_task_specs(int(variant), W, H, pw, ph, None, None, None, 0)
    tt = np.zeros((max(n, 1), 2), np.int32)
    npix = np.zeros(max(n, 1), np.int32)
    lib().ref_make_task_specs(int(variant), W, H, pw, ph, p(tt), p(npix), None, 0)
    total = int(npix[:n].sum())
    pix = np.zeros((max(total, 1), 3), np.int32)
    lib().ref_make_task_specs(int(variant), W, H, pw, ph, p(tt), p(npix), p(pix), total)
    return tt[:n], npix[:n], pix[:total]


def fnv1a64(arr: np.ndarray, h: int = 0xCBF29CE484222325) -> int:
    b = np.ascontiguousarray(arr)
    return int(lib().ref_fnv1a64(p(b), b.nbytes, h))
