"""Round-2 pins of the oracle (CPU only, -m "not gpu"):

* Q29: the oracle's log2-unit FMA exponent against the PLAIN definition
  alpha = min(0.99, o exp(-1/2 d^T Sigma'^-1 d)) (3DGS EWA splatting)
  evaluated in fp64 from the record's conic -- on ~10^5 (conic, d) pairs of
  random anisotropic, rotated Gaussians, within a forward-error bound that
  scales with the exponent's magnitude (a few ulp of alpha for |p| ~ 1).
* O14 (reading Q20): the alpha band, the transmittance band and the a_min band
  flag exactly the constructed near-threshold cases and not their neighbours
  a few band-widths away.
* O12: an INDEPENDENT plain compositor (numpy, fp64, cumulative products; no
  call into the oracle's compositing) over the oracle's records and the
  tile-rectangle rule, on C1 and random tiny scenes -- so the brute force's
  shared composite_pixel is not the only thing pinning the blend.
"""
import math

import numpy as np
import pytest

import synth
from helpers import cam, random_tiny_scene, scene_of

U24 = 2.0 ** -24
LOG2E = 1.4426950408889634
# O14 band constants of the oracle (reading Q20): EX2_REL = 2^-21,
# ALPHA_REL = EX2_REL + 2 U24, safety 2
ALPHA_REL = 2.0 ** -21 + 2 * U24
SAFETY = 2.0
ALPHA_MIN = np.float32(1.0 / 255.0)
CAM = {"fx": 100.0, "fy": 100.0, "cx": 50.0, "cy": 50.0, "width": 100, "height": 100}


def _random_gaussians(rng, n):
    gs = []
    for _ in range(n):
        q = rng.standard_normal(4)
        gs.append({"mu": [rng.uniform(-0.2, 0.2), rng.uniform(-0.2, 0.2), rng.uniform(3.0, 6.0)],
                   "scale": list(np.exp(rng.uniform(math.log(0.02), math.log(0.4), 3))),
                   "quat": list(q / np.linalg.norm(q)), "opacity": float(rng.uniform(0.05, 0.98)),
                   "rgb": [1.0, 1.0, 1.0]})
    return gs


def test_q29_exponent_matches_plain_definition(orc):
    """Single-Gaussian renders with colour 1: the red plane at a pixel is the
    oracle's blend weight w = alpha (T = 1), i.e. its alpha.  Compare with
    min(0.99, o exp(-1/2 (a dx^2 + 2 b dx dy + c dy^2))) in fp64 (conic (a, b, c)
    from the oracle's record).  Bound: |dp| <= 8 U24 S (S = sum of the absolute
    terms of p in log2 units: the oracle's roundings of k, k a, 2k b, k c, the
    products and the two fused adds) -> |dalpha| <= alpha (ln2 |dp| + 2 U24)."""
    rng = np.random.default_rng(2029)
    camera = cam(CAM)
    n_checked = n_zero = 0
    worst = 0.0
    for g in _random_gaussians(rng, 200):
        r = orc.render(scene_of([g]), camera)
        rec = r["rec"]
        if len(rec["gid"]) == 0:
            continue
        a, b, c = (float(x) for x in rec["conic"][0])
        u, v, o = float(rec["u"][0]), float(rec["v"][0]), float(rec["opacity"][0])
        x0, x1, y0, y1 = (int(t) for t in rec["rect"][0])
        ys, xs = np.mgrid[y0 * 16:min(100, y1 * 16 + 16), x0 * 16:min(100, x1 * 16 + 16)]
        dx = np.float32(u) - xs.astype(np.float32)       # the oracle's fp32 offsets (exact inputs)
        dy = np.float32(v) - ys.astype(np.float32)
        dx, dy = dx.astype(np.float64), dy.astype(np.float64)
        power = -0.5 * (a * dx * dx + 2.0 * b * dx * dy + c * dy * dy)
        alpha_def = np.minimum(0.99, o * np.exp(power))
        S = 0.5 * LOG2E * (abs(a) * dx * dx + 2.0 * abs(b) * np.abs(dx * dy) + abs(c) * dy * dy)
        got = r["rgb"][0][ys, xs].astype(np.float64)
        tol = alpha_def * (math.log(2.0) * 8 * U24 * S + 2 * U24) + 1e-12
        clear = np.abs(alpha_def - ALPHA_MIN) > 1e-4 * ALPHA_MIN          # away from the 1/255 cut
        live = clear & (alpha_def >= ALPHA_MIN) & (power <= 0)
        dead = clear & (alpha_def < ALPHA_MIN)
        err = np.abs(got - alpha_def)
        assert (err[live] <= tol[live]).all(), float((err[live] / tol[live]).max())
        assert (got[dead] == 0).all()
        n_checked += int(live.sum())
        n_zero += int(dead.sum())
        small = live & (S <= 1.0)          # |p| <= 1: a few ulp of alpha
        worst = max(worst, float((err[small] / alpha_def[small]).max(initial=0)) / U24)
    assert n_checked > 20000 and n_zero > 20000
    assert worst <= 8.0, worst


def test_q29_wrong_exponent_forms_are_caught(orc):
    """The pin above is sensitive to the plausible mistakes: dropping the factor
    2 of the cross term or the sign of b changes alpha by far more than the bound."""
    rng = np.random.default_rng(7)
    g = _random_gaussians(rng, 1)[0]
    g["scale"] = [0.15, 0.03, 0.08]
    g["quat"] = [0.9, 0.3, 0.2, 0.25]
    r = orc.render(scene_of([g]), cam(CAM))
    a, b, c = (float(x) for x in r["rec"]["conic"][0])
    u, v = float(r["rec"]["u"][0]), float(r["rec"]["v"][0])
    assert abs(b) > 0.05 * math.sqrt(a * c)
    px, py = int(round(u)) + 2, int(round(v)) + 2
    dx, dy = float(np.float32(u) - np.float32(px)), float(np.float32(v) - np.float32(py))
    o = float(r["rec"]["opacity"][0])
    good = min(0.99, o * math.exp(-0.5 * (a * dx * dx + 2 * b * dx * dy + c * dy * dy)))
    bad1 = min(0.99, o * math.exp(-0.5 * (a * dx * dx + b * dx * dy + c * dy * dy)))
    bad2 = min(0.99, o * math.exp(-0.5 * (a * dx * dx - 2 * b * dx * dy + c * dy * dy)))
    got = float(r["rgb"][0, py, px])
    assert abs(got - good) <= 1e-6 * good
    assert abs(got - bad1) > 1e-3 * good and abs(got - bad2) > 1e-3 * good


# ---------------------------------------------------------------- O14 bands (reading Q20)
def _centre(orc, opacity, extra=()):
    """Gaussian(s) exactly at the pixel centre (50, 50): p = 0, alpha_raw = o."""
    gs = [{"mu": [0.0, 0.0, 5.0], "scale": 0.1, "opacity": float(opacity)}]
    gs += [{"mu": [0.0, 0.0, z], "scale": 0.1, "opacity": float(oo)} for z, oo in extra]
    return orc.render(scene_of(gs), cam(CAM), a_min=0.5)


def test_alpha_band_flags_near_cut_only(orc):
    """alpha_raw = o at the centre.  |o - 1/255| <= SAFETY ALPHA_REL o -> flag bit 1;
    four band-widths away -> no flag; the skip decision itself is unchanged.  (Below
    the cut, o < 1/255 is culled as transparent by the projection -- an exact
    input comparison on both sides -- so only o >= 1/255 reaches the band at p = 0.)"""
    band = SAFETY * ALPHA_REL
    for rel, flagged in ((0.0, True), (0.25, True), (0.9, True), (4.0, False), (12.0, False)):
        o = np.float32(float(ALPHA_MIN) * (1.0 + rel * band))
        r = _centre(orc, o)
        assert bool(r["flags"][50, 50] & 1) == flagged, (rel, float(o))
        assert (r["alpha"][50, 50] > 0) == (o >= ALPHA_MIN)


def _t_band(alphas):
    """The band of reading Q20 restated for a sequence of unclamped blends:
    eps_T accumulates ALPHA_REL alpha / (1 - alpha) + 4 U24 per blend."""
    eps = 0.0
    for a in alphas:
        om = np.float32(1.0) - np.float32(a)
        eps += ALPHA_REL * float(a) / float(om) + 4 * U24
    return eps


def test_transmittance_band_flags_near_stop_only(orc):
    """Front layer o1 = 0.98 at the centre leaves T = fl(1 - 0.98); the rear layer's
    o2 is chosen so that T (1 - o2) lands at relative distance rel * band from 1e-4."""
    o1 = np.float32(0.98)
    T1 = np.float32(1.0) - o1
    for rel, flagged in ((0.3, True), (-0.3, True), (5.0, False), (-5.0, False)):
        eps = _t_band([o1]) + ALPHA_REL * 0.99 / 0.01 + 4 * U24    # rear: alpha ~ 0.99
        target = 1e-4 * (1.0 + rel * SAFETY * eps)
        o2 = np.float32(1.0 - target / float(T1))
        if o2 > np.float32(0.99):
            o2 = np.float32(0.99)
        r = _centre(orc, o1, extra=[(10.0, o2)])
        Tn = float(T1 * (np.float32(1.0) - o2))
        real = abs(Tn - 1e-4) / Tn
        eps_here = _t_band([o1]) + ALPHA_REL * float(o2) / float(np.float32(1.0) - o2) + 4 * U24
        expect = real <= SAFETY * eps_here
        assert bool(r["flags"][50, 50] & 2) == expect, (rel, real, eps_here)
        if abs(rel) >= 5.0:
            assert expect == flagged


def test_amin_band_flags_near_threshold_only(orc):
    """One layer at the centre: A = 1 - fl(1 - o).  a_err = SAFETY (T eps_T + 2 U24)
    with eps_T = ALPHA_REL o/(1-o) + 4 U24: flag bit 4 iff |A - a_min| <= a_err."""
    for o, flagged in ((0.5 + 3e-7, True), (0.5 - 3e-7, True), (0.5 + 2e-5, False), (0.5 - 2e-5, False)):
        o = np.float32(o)
        r = _centre(orc, o)
        T = float(np.float32(1.0) - o)
        a_err = SAFETY * (T * (ALPHA_REL * float(o) / T + 4 * U24) + 2 * U24)
        A = float(r["alpha"][50, 50])
        assert abs(r["a_err"][50, 50] - a_err) <= 1e-3 * a_err
        assert bool(r["flags"][50, 50] & 4) == (abs(A - 0.5) <= a_err) == flagged, (float(o), A, a_err)
        assert bool(r["valid"][50, 50]) == (A >= 0.5)


# ---------------------------------------------------------------- independent plain compositor (O12)
def _plain_composite(rec, view, feat=None):
    """The definition of O12 written independently of gs_oracle.cpp: for each pixel
    the Gaussians whose tile rectangle contains its tile, ordered by (depth bits,
    gid); alpha = min(0.99, o exp(power)) in fp64 from the conic; skip power > 0 or
    alpha < 1/255; transmittance by cumulative product; stop before the first
    entry whose T (1 - alpha) < 1e-4.  Returns images and a mask of pixels whose
    decisions are within 1e-5 (relative) of a threshold (excluded)."""
    H, W = view.height, view.width
    u, v, z = (rec[k].astype(np.float64) for k in ("u", "v", "z"))
    a, b, c = (rec["conic"][:, i].astype(np.float64) for i in range(3))
    o, rgb, rect = rec["opacity"].astype(np.float64), rec["rgb"].astype(np.float64), rec["rect"]
    order = np.lexsort((rec["gid"], rec["z"].view(np.uint32)))
    D = 0 if feat is None else feat.shape[1]
    out = dict(rgb=np.zeros((3, H, W)), depth=np.zeros((H, W)), alpha=np.zeros((H, W)), feat=np.zeros((D, H, W)))
    near = np.zeros((H, W), bool)
    for ty in range((H + 15) // 16):
        for tx in range((W + 15) // 16):
            m = order[(rect[order, 0] <= tx) & (tx <= rect[order, 1]) & (rect[order, 2] <= ty) & (ty <= rect[order, 3])]
            for py in range(ty * 16, min(H, ty * 16 + 16)):
                for px in range(tx * 16, min(W, tx * 16 + 16)):
                    if len(m) == 0:
                        continue
                    dx, dy = u[m] - px, v[m] - py
                    power = -0.5 * (a[m] * dx * dx + 2 * b[m] * dx * dy + c[m] * dy * dy)
                    al = np.minimum(0.99, o[m] * np.exp(power))
                    keep = (power <= 0) & (al >= 1.0 / 255.0)
                    amb = np.abs(al - 1.0 / 255.0) <= 1e-5 / 255.0
                    al = np.where(keep, al, 0.0)
                    Tn = np.cumprod(1.0 - al)
                    Tb = np.concatenate([[1.0], Tn[:-1]])
                    stop = np.nonzero(Tn < 1e-4)[0]
                    k = stop[0] if len(stop) else len(m)
                    amb_t = np.abs(Tn[:k + 1] - 1e-4) <= 1e-5 * 1e-4
                    if amb[:k + 1].any() or amb_t.any():
                        near[py, px] = True
                    w = al[:k] * Tb[:k]
                    out["rgb"][:, py, px] = w @ rgb[m[:k]]
                    out["depth"][py, px] = w @ z[m[:k]]
                    out["alpha"][py, px] = 1.0 - (Tb[k] if k < len(m) else Tn[-1])
                    if D:
                        out["feat"][:, py, px] = w @ feat[rec["gid"][m[:k]]].astype(np.float64)
    return out, near


@pytest.mark.parametrize("case", ["C1", "tiny0", "tiny1", "tiny2"])
def test_plain_compositor_agrees_with_oracle(orc, case):
    """O12 against the independent plain compositor: max abs 2e-5 (colour, opacity,
    features), 2e-5 relative (depth) outside the pixels the plain side marks as
    near a threshold (<= 1e-3 of the pixels)."""
    if case == "C1":
        sc, vs = synth.make_config("C1")
        view, feat = vs[0], None
    else:
        rng = np.random.default_rng(int(case[-1]) + 77)
        sc = random_tiny_scene(rng, 150, feat_dim=4 if case == "tiny1" else 0, sh_degree=int(case[-1]) % 4)
        view = synth.make_view(np.eye(3), np.zeros(3), 40.0, 40.0, 23.5, 17.5, 47, 35)
        feat = sc.feat
    r = orc.render(sc, view)
    ref, near = _plain_composite(r["rec"], view, feat)
    ok = ~near
    assert near.mean() <= 1e-3
    assert np.abs(r["rgb"] - ref["rgb"])[:, ok].max() <= 2e-5
    assert np.abs(r["alpha"] - ref["alpha"])[ok].max() <= 2e-5
    dz = np.abs(r["depth"] - ref["depth"])
    assert (dz[ok] <= 2e-5 * np.maximum(np.abs(ref["depth"][ok]), 1e-3)).all()
    if feat is not None:
        assert np.abs(r["feat"] - ref["feat"])[:, ok].max() <= 2e-5 * max(1.0, float(np.abs(feat).max()))
    assert ref["alpha"].max() > 0.5
