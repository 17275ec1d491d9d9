"""CPU: the C-ABI library loads, exports every symbol include/splatsim_b200.h
declares, and its host-only logic (names, statuses, workspace queries,
argument validation, selector, scene synthesis) behaves — no GPU calls."""
from __future__ import annotations

import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle_lib as O
from paper_2412_17378_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "splatsim_b200.h")


def declared_functions() -> list[str]:
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bs_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported():
    L = N.lib()
    names = declared_functions()
    assert len(names) >= 25
    for name in names:
        assert hasattr(L, name), name
    # and the ctypes table covers them all
    assert set(names) <= set(N.SIGNATURES)


def test_no_oracle_in_product_library():
    out = os.popen(f"nm -D {N.LIB_PATH}").read()
    assert "orc_" not in out and "oracle" not in out


def test_versions_and_strings():
    L = N.lib()
    assert L.bs_abi_version() == 1
    assert L.bs_status_string(0) == b"ok"
    assert L.bs_status_string(-2) == b"binning grid does not match image dims"
    for i, name in enumerate(N.VARIANTS):
        assert L.bs_variant_name(i).decode() == name
        assert L.bs_variant_from_name(name.encode()) == i
    assert L.bs_variant_from_name(b"Bogus") == -1
    assert L.bs_variant_name(7) == b"?"


def test_workspace_queries():
    L = N.lib()
    a = L.bs_bin_workspace_bytes(1000, 256, 256, 16, 16, 0)
    b = L.bs_bin_workspace_bytes(1000, 256, 256, 16, 16, 100000)
    c = L.bs_bin_workspace_bytes(100000, 256, 256, 16, 16, 100000)
    assert 0 < a <= b < c  # chunked scatter: no K-sized buffers
    # beyond the chunked path's shared-memory limit the radix path sizes by K
    ra = L.bs_bin_workspace_bytes(1000, 8192, 8192, 16, 16, 0)
    rb = L.bs_bin_workspace_bytes(1000, 8192, 8192, 16, 16, 100000)
    assert 0 < ra < rb
    assert L.bs_bin_workspace_bytes(10, 0, 256, 16, 16, 0) == 0
    assert L.bs_preprocess_workspace_bytes(10**6) > L.bs_preprocess_workspace_bytes(10)
    assert L.bs_tile_stats_workspace_bytes(8160) > 0 and L.bs_render_workspace_bytes(64, 64) >= 64 * 64 * 48 and L.bs_render_workspace_bytes(0, 64) == 0


def test_argument_validation_without_device():
    L = N.lib()
    s = N.Splats(None, None, None)
    cam = N.make_camera(width=64, height=64)
    assert L.bs_preprocess(None, -1, C.byref(cam), s, None, None, 0, None) == -1
    assert L.bs_bin_count(s, 10, None, 64, 64, 16, 16, None, None, 0, None) == -1
    assert L.bs_bin_count(s, 10, None, 64, 64, 0, 16, None, None, 0, None) == -1
    bg = (C.c_float * 3)(0, 0, 0)
    fo = N.FrameOut(None, None, None, None, None, None)
    assert L.bs_render_forward(9, 0, s, None, None, None, 64, 64, 16, 16, bg, fo, None, 0, None) == -1
    assert L.bs_render_forward(0, 5, s, None, None, None, 64, 64, 16, 16, bg, fo, None, 0, None) == -1
    # frames past 2^32 pixels (32-bit pixel indices in the kernels): BS_ERR_UNSUPPORTED before any device work
    one = C.c_void_p(16)
    fo1 = N.FrameOut(one, one, one, one, one, one)
    assert L.bs_render_forward(0, 0, s, None, one, None, 70000, 70000, 32, 32, bg, fo1, None, 0, None) == -6


def test_selector_rule():
    L = N.lib()
    h = N.TileHistogram()
    # balanced 1080p frame: the culled fine-grained kernel still wins on B200
    h.total, h.max, h.tiles, h.mean = 8160 * 1000, 1500, 8160, 1000.0
    assert L.bs_select_variant(C.byref(h), 1920, 1080, 16, 16, 148) == 3
    # one tile dominates the balanced share -> FineGrainedCombined
    h.max = 200000
    assert L.bs_select_variant(C.byref(h), 1920, 1080, 16, 16, 148) == 3
    # (almost) no work: the fixed queue cost loses -> SharedMemOpt
    h.total, h.max, h.tiles, h.mean = 200, 2, 8160, 200 / 8160
    assert L.bs_select_variant(C.byref(h), 1920, 1080, 16, 16, 148) == 4
    assert L.bs_select_variant(None, 1920, 1080, 16, 16, 148) == -1
    # short lists (mean < 12 entries per tile, even with a 30x imbalance):
    # SharedMemOpt (profiles/r2_selector_sweep.jsonl: 1k-Gaussian 1080p / 4K frames)
    h.total, h.max, h.tiles, h.mean = 8160 * 5, 163, 8160, 5.0
    assert L.bs_select_variant(C.byref(h), 1920, 1080, 16, 16, 148) == 4
    h.total, h.max, h.tiles, h.mean = 8160 * 53, 1493, 8160, 53.0  # 10k clustered: FG
    assert L.bs_select_variant(C.byref(h), 1920, 1080, 16, 16, 148) == 3


@pytest.mark.parametrize("n,W,H,f,bgf", [(3000, 1920, 1080, 1000.0, 0.12), (2000, 256, 256, 256.0, 1.0)])
def test_host_generator_matches_oracle(n, W, H, f, bgf):
    ocam = O.make_camera(focal=(f, f), width=W, height=H)
    ref = O.gen_clustered_scene(n, ocam, bgfrac=bgf)
    cam = N.Camera.from_buffer_copy(bytes(ocam))
    got = np.zeros(n, dtype=N.G3D_DTYPE)
    assert N.lib().bs_host_gen_clustered_scene(n, 4, 42, 0.035, bgf, C.byref(cam), got.ctypes.data) == 0
    assert got.tobytes() == ref.tobytes()
