"""CPU-side checks of the C ABI: the library builds, loads without a GPU,
exports every symbol include/gs.h declares, and its host-only entry points
(defaults, batch layout, workspace sizes, argument validation) behave."""
import ctypes
import os
import re

import numpy as np
import pytest

import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def G():
    from paper_2507_15683_b200 import build as B
    B.build()
    import paper_2507_15683_b200 as G
    return G


def declared_functions():
    src = open(os.path.join(ROOT, "include", "gs.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gs_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_four_calls():
    names = declared_functions()
    for f in ("gs_project", "gs_bin_sort", "gs_rasterize", "gs_backproject"):
        assert f in names


def test_library_exports_every_declared_symbol(G):
    L = G.lib()
    for name in declared_functions():
        assert hasattr(L, name), name
    assert set(G.EXPORTS) == set(declared_functions())


def test_abi_version_and_defaults(G):
    L = G.lib()
    assert L.gs_abi_version() == 2
    p = G.default_params()
    import oracle
    o = oracle.Params()
    for k in ("z_near", "dilation", "clamp_margin", "alpha_min", "alpha_max", "t_min"):
        assert getattr(p, k) == np.float32(getattr(o, k)), k


def test_struct_sizes_match_header(G):
    assert ctypes.sizeof(G.gs.gs_view) == 88
    assert ctypes.sizeof(G.gs.gs_scene) == 96
    assert ctypes.sizeof(G.gs.gs_params) == 24
    assert G.gs.RECORD_BYTES == 64


def test_views_layout_contiguous(G):
    L = G.lib()
    vs = synth.pyramid_views(synth.c2_view())
    arr = (G.gs.gs_view * len(vs))()
    for i, v in enumerate(vs):
        arr[i].width, arr[i].height = v.width, v.height
        arr[i].fx = arr[i].fy = 1.0
    tp, tt = ctypes.c_int64(), ctypes.c_int64()
    assert L.gs_views_layout(arr, len(vs), ctypes.byref(tp), ctypes.byref(tt)) == 0
    pix = tiles = 0
    for i, v in enumerate(vs):
        assert arr[i].pix_offset == pix and arr[i].tile_offset == tiles
        pix += v.width * v.height
        tiles += ((v.width + 15) // 16) * ((v.height + 15) // 16)
    assert tp.value == pix and tt.value == tiles
    arr[1].width = 0
    assert L.gs_views_layout(arr, len(vs), ctypes.byref(tp), ctypes.byref(tt)) == 1
    assert b"bad image size" in L.gs_last_error()


def test_workspace_sizes_monotone(G):
    a = G.gs.bin_sort_workspace_bytes(1000, 100)
    b = G.gs.bin_sort_workspace_bytes(100000, 100)
    assert b > a > 0
    assert G.gs.project_workspace_bytes(0, 1) > 0
    assert G.gs.project_workspace_bytes(1024, 256) >= 1024 * 8 * 4


def test_validation_rejects_bad_arguments_without_touching_device(G):
    """Host-side validation returns INVALID_ARG / UNSUPPORTED before any launch."""
    L = G.lib()
    s = G.gs.gs_scene()
    s.n, s.sh_degree, s.feat_dim = 10, 4, 0
    v = (G.gs.gs_view * 1)()
    v[0].width, v[0].height, v[0].fx, v[0].fy = 8, 8, 1.0, 1.0
    p = G.default_params()
    proj = G.gs.gs_projected()
    st = L.gs_project(ctypes.byref(s), v, ctypes.c_void_p(8), 1, ctypes.byref(p), ctypes.byref(proj), None,
                      ctypes.c_size_t(0), None)
    assert st == 2 and b"sh_degree" in L.gs_last_error()
    s.sh_degree, s.feat_dim = 3, 6
    st = L.gs_project(ctypes.byref(s), v, ctypes.c_void_p(8), 1, ctypes.byref(p), ctypes.byref(proj), None,
                      ctypes.c_size_t(0), None)
    assert st == 2 and b"feat_dim" in L.gs_last_error()
    st = L.gs_backproject(None, v, ctypes.c_void_p(8), 1, ctypes.c_float(0.5), None, None, None)
    assert st == 1
    # the fused raster + back-projection: NULL xyz / valid and a NaN a_min are rejected up front
    s.feat_dim = 0
    st = L.gs_rasterize_backproject(ctypes.byref(s), None, None, v, ctypes.c_void_p(8), 1, ctypes.byref(p), None,
                                    ctypes.c_float(0.5), None, None, None)
    assert st == 1 and b"xyz" in L.gs_last_error()
    st = L.gs_rasterize_backproject(ctypes.byref(s), None, None, v, ctypes.c_void_p(8), 1, ctypes.byref(p), None,
                                    ctypes.c_float(float("nan")), ctypes.c_void_p(16), ctypes.c_void_p(16), None)
    assert st == 1 and b"a_min" in L.gs_last_error()


def test_no_cpu_fallback_in_product_path():
    """The product package never imports the oracle (it must fail loudly
    without its CUDA library instead of falling back)."""
    pkg = os.path.join(ROOT, "paper_2507_15683_b200")
    for f in os.listdir(pkg):
        if f.endswith(".py"):
            txt = open(os.path.join(pkg, f)).read()
            assert "import oracle" not in txt and "from oracle" not in txt, f


def test_new_calls_validate_on_the_host(G):
    """gs_match / gs_pnp / gs_verify_consistency / gs_validate_scene /
    gs_scene_features_f16 reject bad arguments before any launch (no GPU needed)."""
    L = G.lib()
    fake = ctypes.c_void_p(256)
    m = G.gs.gs_matches()
    # NULL outputs
    st = L.gs_match(fake, fake, 1, 32, 64, 64, ctypes.c_float(0.1), ctypes.c_float(0.05), None, None, fake,
                    ctypes.c_size_t(1 << 30), ctypes.byref(m), None)
    assert st == 1 and b"NULL" in L.gs_last_error()
    m.coarse = m.coarse_prob = m.peak = m.prob = m.ref = fake
    st = L.gs_match(fake, fake, 1, 24, 64, 64, ctypes.c_float(0.1), ctypes.c_float(0.05), None, None, fake,
                    ctypes.c_size_t(1 << 30), ctypes.byref(m), None)
    assert st == 2 and b"D = 24" in L.gs_last_error()                 # UNSUPPORTED feature width
    st = L.gs_match(fake, fake, 1, 32, 60, 64, ctypes.c_float(0.1), ctypes.c_float(0.05), None, None, fake,
                    ctypes.c_size_t(1 << 30), ctypes.byref(m), None)
    assert st == 1 and b"multiples of 8" in L.gs_last_error()
    st = L.gs_match(fake, fake, 1, 32, 64, 64, ctypes.c_float(0.0), ctypes.c_float(0.05), None, None, fake,
                    ctypes.c_size_t(1 << 30), ctypes.byref(m), None)
    assert st == 1 and b"tau" in L.gs_last_error()
    need = G.match_workspace_bytes(1, 32, 64, 64)
    st = L.gs_match(fake, fake, 1, 32, 64, 64, ctypes.c_float(0.1), ctypes.c_float(0.05), None, None, fake,
                    ctypes.c_size_t(need - 1), ctypes.byref(m), None)
    assert st == 3                                                      # WORKSPACE_TOO_SMALL
    stats = ctypes.c_void_p(512)
    st = L.gs_pnp(fake, fake, 1, 8, 8, fake, ctypes.c_float(3.0), 999, 0, 1024, fake, ctypes.c_size_t(1 << 30),
                  ctypes.c_void_p(1024), stats, None)
    assert st == 2 and b"n_hyp" in L.gs_last_error()
    st = L.gs_pnp(fake, fake, 1, 8, 8, fake, ctypes.c_float(3.0), 64, 0, 1024, fake, ctypes.c_size_t(1 << 30),
                  fake, stats, None)
    assert st == 1 and b"alias" in L.gs_last_error()
    st = L.gs_pnp(fake, fake, 1, 8, 8, fake, ctypes.c_float(3.0), 64, 0, 1024, fake, ctypes.c_size_t(16),
                  ctypes.c_void_p(1024), stats, None)
    assert st == 3
    st = L.gs_verify_consistency(fake, 3, 1, ctypes.c_float(20.0), None, None, fake, None)
    assert st == 1
    s = G.gs.gs_scene()
    s.n, s.sh_degree, s.feat_dim = 10, 0, 0
    st = L.gs_validate_scene(ctypes.byref(s), 0, None, None, None)
    assert st == 1                                                      # geometry pointers NULL
    st = L.gs_scene_features_f16(ctypes.byref(s), fake, None)
    assert st == 1 and b"no features" in L.gs_last_error()
    assert G.match_workspace_bytes(0, 32, 64, 64) == 0 and G.pnp_workspace_bytes(0, 10) == 0


def test_struct_sizes_of_n2_types(G):
    assert ctypes.sizeof(G.gs.gs_matches) == 7 * 8
    assert ctypes.sizeof(G.gs.gs_pnp_stats) == 16
    assert ctypes.sizeof(G.gs.gs_bins) == 8 * 7 + 8


def test_dssim_validates_on_the_host(G):
    """gs_dssim_grad (Eq. 3's D-SSIM) rejects bad arguments before any launch; empty
    input is a no-op; the workspace is three fp32 planes per input plane."""
    L = G.lib()
    fake = ctypes.c_void_p(256)
    one = ctypes.c_float(1.0)
    assert G.lib().gs_dssim_workspace_bytes(3, 768, 1024) == 3 * 3 * 768 * 1024 * 4
    assert G.lib().gs_dssim_workspace_bytes(0, 768, 1024) == 0
    assert L.gs_dssim_grad(fake, fake, -1, 4, 4, one, fake, fake, ctypes.c_size_t(1 << 20), fake, None) == 1
    assert L.gs_dssim_grad(fake, fake, 70000, 4, 4, one, fake, fake, ctypes.c_size_t(1 << 30), fake, None) == 1
    assert L.gs_dssim_grad(fake, None, 1, 4, 4, one, fake, fake, ctypes.c_size_t(1 << 20), fake, None) == 1
    assert b"NULL" in L.gs_last_error()
    assert L.gs_dssim_grad(fake, fake, 2, 4, 4, one, fake, fake, ctypes.c_size_t(2 * 3 * 16 * 4 - 1), fake,
                           None) == 3
    assert L.gs_dssim_grad(None, None, 0, 4, 4, one, None, None, ctypes.c_size_t(0), None, None) == 0
