"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs.  Bit-exact records / keys / ranges; images within the
north_star tolerances (tests/parity.py).  All tests need a B200."""
import dataclasses
import math

import numpy as np
import pytest

import synth
from helpers import random_tiny_scene, scene_of
import parity as PT

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def G():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2507_15683_b200 as G
    G.lib()
    return G


def _gpu_render(G, scene, views, use_blocks=True, debug_keys=True, feat=True, f16=True, **kw):
    ds = G.DeviceScene(scene, use_f16_features=f16)
    r = G.Renderer(ds, views, debug_keys=debug_keys, use_blocks=use_blocks, **kw)
    r.render()
    torch.cuda.synchronize()
    return r


def compare_view(G, r, i, scene, view, orc, check_bp=True, report=None):
    cap = r.proj.rec_capacity
    n = min(int(r.proj.n_rec[i].item()), cap)
    recs = PT.decode_records(r.proj.records()[i * cap:i * cap + n].cpu().numpy())
    PT.check_records(recs, orc["rec"], i)
    TX, TY = (view.width + 15) // 16, (view.height + 15) // 16
    t0 = r.vb.tile_offset(i)
    rg = r.bins.ranges.view(-1, 2)[t0:t0 + TX * TY].cpu().numpy().view(np.uint32)
    s0, s1 = int(rg[0, 0]), int(rg[-1, 1])
    sorted_rec = r.bins.sorted_rec[s0:s1].cpu().numpy().view(np.uint32).astype(np.int64)
    idx = sorted_rec - i * cap
    assert ((idx >= 0) & (idx < n)).all(), "pair points outside its view's records"
    tiles = np.repeat(np.arange(TX * TY, dtype=np.uint32), (rg[:, 1] - rg[:, 0]).astype(np.int64))
    gk = (tiles, recs["z"][idx].view(np.uint32), recs["gid"][idx], (rg.astype(np.int64) - s0).astype(np.uint32))
    PT.check_keys(gk, orc["keys"])
    if r.bins.sorted_key is not None:
        sk = r.bins.sorted_key[s0:s1].cpu().numpy().view(np.uint64)
        np.testing.assert_array_equal((sk >> np.uint64(32)).astype(np.uint32) - np.uint32(t0), orc["keys"]["tile"])
        np.testing.assert_array_equal((sk & np.uint64(0xFFFFFFFF)).astype(np.uint32), orc["keys"]["depth"])
    img = {k: v.cpu().numpy() for k, v in r.view_images(i).items()}
    stats = PT.check_images(img, orc, report=report)
    if check_bp and "xyz" in img and "xyz" in orc:
        PT.check_backproject(img["xyz"], img["valid"], orc["xyz"], orc["valid"], orc["flags"], orc["depth"],
                             orc["alpha"])
    return stats


# ------------------------------------------------------------------ C1 + tiny
def test_c1_full_parity(G, orc):
    sc, vs = synth.make_config("C1")
    r = _gpu_render(G, sc, vs)
    o = orc.render(sc, vs[0], a_min=0.5, binning="tight")
    PT.assert_flag_budget([compare_view(G, r, 0, sc, vs[0], o)])


def test_c1_features_D8(G, orc):
    sc = synth.box_v1(1000, seed=11, feat_dim=8)
    v = synth.box_view()
    r = _gpu_render(G, sc, [v])
    o = orc.render(sc, v, a_min=0.5, binning="tight")
    PT.assert_flag_budget([compare_view(G, r, 0, sc, v, o)])


@pytest.mark.parametrize("seed", range(12))
def test_random_tiny_ragged(G, orc, seed):
    """Ragged image sizes (partial edge tiles), behind-camera / off-screen /
    transparent Gaussians, depth ties, un-normalised q, SH 0-3, D in {0, 4, 12}."""
    rng = np.random.default_rng(500 + seed)
    D = [0, 4, 12][seed % 3]
    sc = random_tiny_scene(rng, int(rng.integers(20, 400)), feat_dim=D, sh_degree=seed % 4)
    W, H = int(rng.integers(1, 90)), int(rng.integers(1, 70))
    v = synth.make_view(np.eye(3), np.zeros(3), 40.0, 40.0, W / 2 - 0.5, H / 2 - 0.5, W, H)
    r = _gpu_render(G, sc, [v])
    o = orc.render(sc, v, a_min=0.5, binning="tight")
    PT.assert_flag_budget([compare_view(G, r, 0, sc, v, o)])


@pytest.mark.parametrize("D,seed", [(16, 0), (32, 1), (48, 2), (64, 3), (32, 4), (16, 5)])
def test_feature_contraction_tcgen05_and_mma_sync(G, orc, D, seed):
    """Feature blend F = sum_k w_k f_k on both tensor-core paths:
    tcgen05 (fp16 feature rows, TMEM accumulators; D in {16, 32, 48, 64}) and
    mma.sync (fp32 rows).  Both against the oracle, ragged image sizes."""
    rng = np.random.default_rng(1300 + seed)
    sc = random_tiny_scene(rng, int(rng.integers(100, 600)), feat_dim=D, sh_degree=seed % 4)
    W, H = int(rng.integers(20, 120)), int(rng.integers(10, 90))
    v = synth.make_view(np.eye(3), np.zeros(3), 40.0, 40.0, W / 2 - 0.5, H / 2 - 0.5, W, H)
    o = orc.render(sc, v, a_min=0.5, binning="tight")
    feats, st = [], []
    for f16 in (True, False):
        r = _gpu_render(G, sc, [v], f16=f16)
        st.append(compare_view(G, r, 0, sc, v, o))
        feats.append(r.view_images(0)["feat"].clone())
    PT.assert_flag_budget(st)
    # same fp16-rounded features and hi+lo weights: the paths differ by fp32 summation order only
    scale = max(1.0, float(np.abs(sc.feat).max()))
    assert float((feats[0] - feats[1]).abs().max()) <= 1e-4 * scale


def test_empty_scene(G, orc):
    sc = scene_of([])
    v = synth.box_view()
    r = _gpu_render(G, sc, [v])
    img = r.view_images(0)
    assert not img["rgb"].any() and not img["alpha"].any() and not img["depth"].any()
    assert not img["valid"].any()


def test_all_culled(G, orc):
    sc = scene_of([{"mu": [0, 0, -5]}, {"mu": [100, 0, 5]}, {"mu": [0, 0, 5], "opacity": 0.001}])
    v = synth.box_view()
    r = _gpu_render(G, sc, [v])
    assert int(r.proj.n_rec[0]) == 0 and r.n_pairs() == 0
    d = r.proj.diag.cpu().numpy()
    assert list(d) == [1, 1, 0, 1]
    assert not r.view_images(0)["alpha"].any()


def test_diag_counters_match_oracle(G, orc):
    sc = scene_of([{"mu": [0, 0, 5], "scale": [0.1, 0.0, 0.1]}, {"mu": [0, 0, 5], "opacity": 0.001},
                   {"mu": [-10.0, 0, 5], "scale": 0.01}, {"mu": [0, 0, 0.1]}, {"mu": [0, 0, 5], "quat": [0, 0, 0, 0]},
                   {"mu": [0, 0, 5]}])
    v = synth.make_view(np.eye(3), np.zeros(3), 100, 100, 50, 50, 100, 100)
    r = _gpu_render(G, sc, [v])
    o = orc.project(sc, v)
    d = r.proj.diag.cpu().numpy()
    assert list(d) == [o["diag"]["near"], o["diag"]["transparent"], o["diag"]["degenerate"], o["diag"]["offscreen"]]


def test_overflow_then_recovery(G, orc):
    """Tiny capacities set the status bits; Renderer.render re-runs with the
    sizes the device reported and then matches the oracle."""
    sc, vs = synth.make_config("C1")
    ds = G.DeviceScene(sc)
    r = G.Renderer(ds, vs, rec_capacity=16, pair_capacity=64, debug_keys=True)
    r.run()
    assert r.status() & 1
    r.render()
    assert r.status() == 0
    o = orc.render(sc, vs[0], a_min=0.5, binning="tight")
    PT.assert_flag_budget([compare_view(G, r, 0, sc, vs[0], o)])
    r2 = G.Renderer(ds, vs, pair_capacity=64)
    r2.run()
    assert r2.status() == 2 and r2.n_pairs() == len(o["keys"]["tile"])


# ------------------------------------------------------------------ aerial configs
def test_c2_full_size_parity(G, orc):
    """C2 at its BASELINE size (200k Gaussians, SH 3, 1024x768): whole image."""
    sc, vs = synth.make_config("C2")
    r = _gpu_render(G, sc, vs)
    o = orc.render(sc, vs[0], a_min=0.5, binning="tight")
    st = compare_view(G, r, 0, sc, vs[0], o)
    print("C2 stats", st)
    PT.assert_flag_budget([st])


def test_c2_blocks_do_not_change_result(G, orc):
    sc, vs = synth.make_config("C2", scale=0.25)
    a = _gpu_render(G, sc, vs, use_blocks=True)
    b = _gpu_render(G, sc, vs, use_blocks=False)
    for k in ("rgb", "depth", "alpha"):
        assert torch.equal(a.view_images(0)[k], b.view_images(0)[k])


def test_c3_pyramid_parity(G, orc):
    """C3 shape (5-level pyramid 64x48 -> 1024x768, D = 32, SH 3) at reduced N;
    each level against the oracle; level 4 == the same camera rendered alone
    (batching invariance, Q21)."""
    sc, vs = synth.make_config("C3", scale=0.02)
    r = _gpu_render(G, sc, vs)
    st = []
    for i, v in enumerate(vs):
        o = orc.render(sc, v, a_min=0.5, binning="tight")
        st.append(compare_view(G, r, i, sc, v, o))
    PT.assert_flag_budget(st)
    alone = _gpu_render(G, sc, [vs[-1]])
    for k in ("rgb", "depth", "alpha", "feat"):
        assert torch.equal(alone.view_images(0)[k], r.view_images(len(vs) - 1)[k])


def test_c3_coarse_level_long_lists(G, orc):
    """Coarse pyramid level with very long tile lists (> 8192 entries per tile):
    exercises the shared-memory bitonic + merge-path path of gs_bin_sort.  The
    whole pyramid (level 0 = the long lists) is compared; the flag budget is
    over its 1,047,552 pixels."""
    sc, vs = synth.make_config("C3", scale=0.1)
    r = _gpu_render(G, sc, vs)
    st = []
    for i, v in enumerate(vs):
        o = orc.render(sc, v, a_min=0.5, binning="tight")
        if i == 0:
            rg = o["keys"]["ranges"]
            assert (rg[:, 1] - rg[:, 0]).max() > 8192
        st.append(compare_view(G, r, i, sc, v, o))
    PT.assert_flag_budget(st)


def test_c3_full_size_parity(G, orc):
    """C3 at its BASELINE size (2M Gaussians, SH 3, D = 32, the 5-level pyramid
    64x48 -> 1024x768 rendered in one batch, P:276 H_f/H_c = 8): every level whole
    against the oracle, keys bit-exact, flag budget over all 1,047,552 pixels."""
    sc, vs = synth.make_config("C3")
    r = _gpu_render(G, sc, vs, debug_keys=False)
    st = []
    for i, v in enumerate(vs):
        o = orc.render(sc, v, a_min=0.5, binning="tight")
        st.append(compare_view(G, r, i, sc, v, o))
    PT.assert_flag_budget(st)


def test_c4_batch_parity_and_invariance(G, orc):
    """C4 shape (256-pose grid, D = 32) at reduced N: 6 views of the batch vs
    the oracle; a view rendered inside the batch equals the view alone."""
    sc, vs = synth.make_config("C4", scale=0.02)
    vs = vs[:24]
    r = _gpu_render(G, sc, vs)
    st = []
    for i in (0, 5, 11, 17, 23):
        o = orc.render(sc, vs[i], a_min=0.5, binning="tight")
        st.append(compare_view(G, r, i, sc, vs[i], o))
    PT.assert_flag_budget(st)
    alone = _gpu_render(G, sc, [vs[11]])
    for k in ("rgb", "depth", "alpha", "feat", "xyz", "valid"):
        assert torch.equal(alone.view_images(0)[k], r.view_images(11)[k])


def test_c5_oblique_parity(G, orc):
    """C5 shape (oblique 1920x1080, 8 blocks, backprojection) at reduced N."""
    sc, vs = synth.make_config("C5", scale=0.005)
    vs = vs[:4]
    r = _gpu_render(G, sc, vs)
    st = []
    for i in (0, 3):
        o = orc.render(sc, vs[i], a_min=0.5, binning="tight")
        st.append(compare_view(G, r, i, sc, vs[i], o))
    PT.assert_flag_budget(st)


def test_determinism_run_to_run(G, orc):
    sc, vs = synth.make_config("C4", scale=0.01)
    vs = vs[:8]
    ds = G.DeviceScene(sc)
    r = G.Renderer(ds, vs)
    r.render()
    first = {k: v.clone() for k, v in r.view_images(3).items()}

    def key_gids():
        # record slots depend on atomic order; the (tile, depth, gid) list must not
        recs = r.proj.records()
        return recs[r.bins.sorted_rec[:r.n_pairs()].long(), 12].clone(), r.bins.ranges.clone()

    keys = key_gids()
    for _ in range(3):
        r.run()
        torch.cuda.synchronize()
        for k, v in r.view_images(3).items():
            assert torch.equal(v, first[k]), k
        k2 = key_gids()
        assert torch.equal(keys[0], k2[0]) and torch.equal(keys[1], k2[1])


def test_backproject_kernel_on_oracle_images(G, orc):
    """gs_backproject in isolation: fed the oracle's own depth/alpha planes,
    it must match the oracle's back-projection (|dX| <= 1e-3 scene scale,
    identical valid masks except flagged pixels)."""
    sc, vs = synth.make_config("C2", scale=0.25)
    v = vs[0]
    o = orc.render(sc, v, a_min=0.5, binning="tight")
    vb = G.ViewBatch([v])
    img = G.Images(vb.total_pixels, 0)
    img.depth.copy_(torch.from_numpy(o["depth"].reshape(-1)))
    img.alpha.copy_(torch.from_numpy(o["alpha"].reshape(-1)))
    xyz = torch.empty(3 * vb.total_pixels, device="cuda")
    valid = torch.empty(vb.total_pixels, dtype=torch.uint8, device="cuda")
    G.gs_backproject(img, vb, 0.5, xyz, valid)
    torch.cuda.synchronize()
    H, W = v.height, v.width
    PT.check_backproject(xyz.view(3, H, W).cpu().numpy(), valid.view(H, W).cpu().numpy(), o["xyz"], o["valid"],
                         o["flags"], o["depth"], o["alpha"])


def test_fused_backproject_equals_separate_kernel(G):
    """gs_rasterize_backproject (O13 in the compositing epilogue; the Renderer's
    default) writes exactly what gs_backproject writes from the same images."""
    sc, vs = synth.make_config("C4", scale=0.01)
    vs = vs[:4]
    ds = G.DeviceScene(sc)
    r = G.Renderer(ds, vs)
    r.render()
    torch.cuda.synchronize()
    xyz2 = torch.full_like(r.xyz, float("nan"))
    valid2 = torch.full_like(r.valid, 7)
    G.gs_backproject(r.images, r.vb, r.a_min, xyz2, valid2)
    torch.cuda.synchronize()
    n = r.vb.total_pixels
    assert int(r.valid[:n].sum()) > 0
    assert torch.equal(r.valid[:n], valid2[:n])
    assert torch.equal(r.xyz, xyz2)


# ------------------------------------------------------------------ full-size sampled parity
@pytest.mark.parametrize("cfg,views", [("C4", (0, 37, 74, 111, 137, 180, 222, 255)), ("C5", (0, 9, 33, 63))])
def test_full_size_sampled_views(G, orc, cfg, views):
    """BASELINE sizes in the bench's launch configuration (whole batch in one
    launch of each kernel): sampled views spread over the batch compared whole
    against the oracle (C4: 8 of 256, C5: 4 of 64)."""
    sc, vs = synth.make_config(cfg)
    ds = G.DeviceScene(sc)
    r = G.Renderer(ds, vs, debug_keys=False)
    r.render()
    torch.cuda.synchronize()
    st = []
    for i in views:
        o = orc.render(sc, vs[i], a_min=0.5, binning="tight")
        st.append(compare_view(G, r, i, sc, vs[i], o))
    PT.assert_flag_budget(st)


# ------------------------------------------------------------------ gs_validate_scene (debug, S:90 / S:106)
@pytest.mark.parametrize("field,idx,value,reason", [
    ("pos", 17, np.nan, "position"), ("quat", 3, 0.0, "quat"), ("scale", 40, -1.0, "scale"),
    ("scale", 41, 0.0, "scale"), ("opacity", 9, 1.5, "opacity"), ("opacity", 10, np.nan, "opacity"),
    ("sh", 55, np.inf, "sh"), ("feat", 70, np.nan, "feature")])
def test_validate_scene_names_first_offender(G, field, idx, value, reason):
    sc = synth.box_v1(200, seed=3, feat_dim=8, sh_degree=1)
    ds = G.DeviceScene(sc)
    assert G.gs_validate_scene(ds) == (-1, "none")
    arr = getattr(sc, field).copy()
    for i in (idx, idx + 100):                  # two offenders: the first is reported
        if field == "quat":
            arr[:, i] = value                   # zero quaternion
        elif field == "feat":
            arr[i, 1] = value
        elif arr.ndim == 2:
            arr[-1, i] = value                  # last component / coefficient of Gaussian i
        else:
            arr[i] = value
    bad = dataclasses.replace(sc, **{field: arr})
    assert G.gs_validate_scene(G.DeviceScene(bad)) == (idx, reason)


def test_validate_scene_unit_quaternion_mode(G):
    """S:90 requires |q| = 1 within 1e-6; the hot path normalises (Q2), so that
    check is opt-in."""
    sc = synth.box_v1(50, seed=4)
    q = sc.quat.copy()
    q /= np.linalg.norm(q, axis=0, keepdims=True)
    q[:, 12] *= 1.001
    bad = dataclasses.replace(sc, quat=q.astype(np.float32))
    ds = G.DeviceScene(bad)
    assert G.gs_validate_scene(ds) == (-1, "none")
    assert G.gs_validate_scene(ds, unit_quat=True) == (12, "quat_norm")


# ------------------------------------------------------------------ N3: binning modes
@pytest.mark.parametrize("cfg,scale,nv", [("C2", 0.25, 1), ("C4", 0.01, 4), ("C5", 0.005, 2)])
def test_square_and_tight_binning_keys_and_identical_images(G, orc, cfg, scale, nv):
    """GS_BIN_SQUARE keys bit-exact against the oracle's square mode, GS_BIN_TIGHT
    keys against its tight mode (reading Q30); the two modes render bit-identical
    RGB, depth, opacity, back-projection and contributions on the GPU (features
    up to fp32 summation grouping)."""
    sc, vs = synth.make_config(cfg, scale=scale)
    vs = vs[:nv]
    rs = {b: _gpu_render(G, sc, vs, binning=b, contrib=True) for b in ("square", "tight")}
    assert rs["tight"].n_pairs() < rs["square"].n_pairs()
    st = []
    for i in range(nv):
        for b, r in rs.items():
            o = orc.render(sc, vs[i], a_min=0.5, binning=b)
            st.append(compare_view(G, r, i, sc, vs[i], o))
        a, b = rs["square"].view_images(i), rs["tight"].view_images(i)
        for k in ("rgb", "depth", "alpha", "xyz", "valid"):
            assert torch.equal(a[k], b[k]), k
        if "feat" in a:
            # same blends; a zero-weight row the warp cull admits only in square mode shifts
            # the grouping of the tensor-core k-steps, i.e. the fp32 summation order
            scale = max(1.0, float(np.abs(sc.feat).max()))
            assert float((a["feat"] - b["feat"]).abs().max()) <= 1e-5 * scale
    assert torch.equal(rs["square"].proj.contrib.sum(), rs["tight"].proj.contrib.sum())
    PT.assert_flag_budget(st)


def test_pack_images_compact_transport(G):
    """gs_pack_images (reading Q39): per view at byte 12 * pix_offset, fp16 R, G, B, A
    planes equal to the fp32 images rounded to nearest, then the fp32 depth plane
    bit-identical; views of different sizes (the C3 pyramid) and an odd-sized view."""
    sc, vs = synth.make_config("C3", scale=0.02)
    odd = synth.make_view(vs[0].R, vs[0].t, vs[0].fx, vs[0].fy, 30.0, 20.0, 61, 41)
    views = vs + [odd]
    r = _gpu_render(G, sc, views)
    n = r.vb.total_pixels
    out = torch.zeros(12 * n + 16, dtype=torch.uint8, device="cuda")
    G.gs_pack_images(r.images, r.vb, out)
    torch.cuda.synchronize()
    buf = out.cpu().numpy()
    for i, v in enumerate(views):
        hw, po = v.width * v.height, r.vb.pix_offset(i)
        blk = buf[12 * po:12 * (po + hw)]
        halves = blk[:8 * hw].view(np.float16).reshape(4, hw)
        depth = blk[8 * hw:].view(np.float32)
        img = {k: t.cpu().numpy() for k, t in r.view_images(i).items()}
        np.testing.assert_array_equal(halves[:3], img["rgb"].reshape(3, hw).astype(np.float16))
        np.testing.assert_array_equal(halves[3], img["alpha"].reshape(hw).astype(np.float16))
        np.testing.assert_array_equal(depth, img["depth"].reshape(hw))
        assert np.abs(halves[:3].astype(np.float32) - img["rgb"].reshape(3, hw)).max() <= 1e-3


def test_pack_images_dense11_transport(G):
    """GS_PACK_DENSE11 (reading Q39): batch-planar fp16 R, G, B (= the fp32 images rounded
    to nearest), unorm16 A (|error| <= 0.5/65535) and the depth plane's upper 24 bits
    (relative error <= 2^-16); host decode with unpack_dense11; pyramid + odd-sized view
    (the scalar tail) and a 4-aligned batch (the vector path)."""
    for cfg, extra in (("C3", True), ("C2", False)):
        sc, vs = synth.make_config(cfg, scale=0.02 if cfg == "C3" else 0.05)
        views = list(vs)
        if extra:
            views.append(synth.make_view(vs[0].R, vs[0].t, vs[0].fx, vs[0].fy, 30.0, 20.0, 61, 41))
        r = _gpu_render(G, sc, views)
        n = r.vb.total_pixels
        assert G.gs_pack_bytes(n, G.GS_PACK_DENSE11) == 11 * n
        out = torch.zeros(11 * n + 16, dtype=torch.uint8, device="cuda")
        G.gs_pack_images(r.images, r.vb, out, fmt=G.GS_PACK_DENSE11)
        torch.cuda.synchronize()
        rgb, depth, alpha = G.unpack_dense11(out.cpu().numpy(), n)
        for i, v in enumerate(views):
            hw, po = v.width * v.height, r.vb.pix_offset(i)
            img = {k: t.cpu().numpy() for k, t in r.view_images(i).items()}
            ref_rgb = img["rgb"].reshape(3, hw)
            np.testing.assert_array_equal(rgb[:, po:po + hw], ref_rgb.astype(np.float16).astype(np.float32))
            a = img["alpha"].reshape(hw).astype(np.float64)
            assert np.abs(alpha[po:po + hw] - a).max() <= 0.5 / 65535 + 1e-7
            z = img["depth"].reshape(hw).astype(np.float64)
            dz = np.abs(depth[po:po + hw].astype(np.float64) - z)
            assert (dz <= z * 2.0 ** -16 + 1e-30).all(), dz.max()

