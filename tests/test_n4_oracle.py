"""Pins of the oracle's N4 row: the feature-field backward of
Eq. 2 with the geometry frozen, dL/df_g = sum_px w_g(px) dL/dF(px).
Pins: exact linearity (a finite difference of the linear loss <g, F(f)> in f
equals the gradient to fp64 rounding), the sum identity sum_g dL/df_g = sum_px
A(px) g(px) (sum_k w_k = A), and binning-mode invariance."""
import dataclasses

import numpy as np
import pytest

import synth
from helpers import random_tiny_scene


def _setup(orc, seed, D=8, binning="square"):
    rng = np.random.default_rng(seed)
    sc = random_tiny_scene(rng, 120, feat_dim=D)
    v = synth.make_view(np.eye(3), np.zeros(3), 40.0, 40.0, 23.5, 17.5, 48, 36)
    o = orc.render(sc, v, binning=binning)
    g = rng.standard_normal((D, v.height, v.width))
    return rng, sc, v, o, g


@pytest.mark.parametrize("seed", range(4))
def test_feature_grad_equals_finite_difference_of_linear_loss(orc, seed):
    rng, sc, v, o, g = _setup(orc, seed)
    grad = orc.feature_grad(v, o["rec"], o["keys"], sc.feat, g.astype(np.float32), sc.n)
    g32 = g.astype(np.float32).astype(np.float64)
    loss = lambda F: float((F.astype(np.float64) * g32).sum())
    base = loss(o["feat"])
    hit = np.nonzero(np.abs(grad).sum(1) > 0)[0]
    assert len(hit) > 5
    for gi in rng.choice(hit, 5, replace=False):
        c = int(rng.integers(sc.feat_dim))
        f2 = sc.feat.copy()
        f2[gi, c] += 0.5                                   # exact in fp32 for |f| < 2^22
        import dataclasses
        o2 = orc.render(dataclasses.replace(sc, feat=f2), v)
        # the rendered map is stored in fp32: allow its rounding
        fd = (loss(o2["feat"]) - base) / 0.5
        assert abs(fd - grad[gi, c]) <= 1e-4 * max(1.0, abs(grad[gi, c])) + 1e-4 * np.abs(g32).sum() * 1e-3


@pytest.mark.parametrize("seed", range(3))
def test_feature_grad_sums_to_alpha_weighted_upstream(orc, seed):
    _, sc, v, o, g = _setup(orc, 10 + seed)
    grad = orc.feature_grad(v, o["rec"], o["keys"], sc.feat, g.astype(np.float32), sc.n)
    expect = (o["alpha"].astype(np.float64)[None] * g.astype(np.float32).astype(np.float64)).sum((1, 2))
    np.testing.assert_allclose(grad.sum(0), expect, rtol=1e-5, atol=1e-6)


def test_feature_grad_same_in_square_and_tight_binning(orc):
    _, sc, v, o, g = _setup(orc, 20)
    a = orc.feature_grad(v, o["rec"], o["keys"], sc.feat, g.astype(np.float32), sc.n)
    o2 = orc.render(sc, v, binning="tight")
    b = orc.feature_grad(v, o2["rec"], o2["keys"], sc.feat, g.astype(np.float32), sc.n)
    np.testing.assert_array_equal(a, b)


# ------------------------------------------------------------------ radiance backward
K2 = np.float32(-0.72134752044448170368)


def _loss(orc, v, rec, keys, gC, gD, gA):
    return orc.radiance_backward(v, rec, keys, gC, gD, gA)[1]


@pytest.mark.parametrize("seed", range(3))
def test_radiance_grad_rgb_and_depth_exact_linearity(orc, seed):
    """C and Dz are linear in each record's rgb and z (weights unaffected):
    central differences equal the gradient on any scene."""
    rng = np.random.default_rng(60 + seed)
    sc = random_tiny_scene(rng, 150, sh_degree=seed % 4)
    v = synth.make_view(np.eye(3), np.zeros(3), 40.0, 40.0, 23.5, 17.5, 48, 36)
    o = orc.render(sc, v)
    rec, keys = o["rec"], o["keys"]
    gC = rng.standard_normal((3, 36, 48)).astype(np.float32)
    gD = rng.standard_normal((36, 48)).astype(np.float32)
    gA = rng.standard_normal((36, 48)).astype(np.float32)
    grad, _ = orc.radiance_backward(v, rec, keys, gC, gD, gA)
    hit = np.nonzero(np.abs(grad[:, 6:]).sum(1) > 0)[0]
    assert len(hit) > 5
    for i in rng.choice(hit, 5, replace=False):
        for f, (field, col) in enumerate((("rgb", 0), ("rgb", 1), ("rgb", 2), ("z", None))):
            r2 = {k: np.array(a, copy=True) for k, a in rec.items() if isinstance(a, np.ndarray)}
            r3 = {k: np.array(a, copy=True) for k, a in rec.items() if isinstance(a, np.ndarray)}
            h = 0.25
            if col is None:
                r2[field][i] += h; r3[field][i] -= h
            else:
                r2[field][i, col] += h; r3[field][i, col] -= h
            fd = (_loss(orc, v, r2, keys, gC, gD, gA) - _loss(orc, v, r3, keys, gC, gD, gA)) / (2 * h)
            np.testing.assert_allclose(fd, grad[i, 6 + f], rtol=1e-6, atol=1e-9)


def _smooth_fixture():
    """Three large layered Gaussians over a 24x20 image: no alpha >= 1/255 boundary,
    clamp or stop crosses a pixel under small perturbations -- the loss is smooth."""
    from helpers import scene_of
    sc = scene_of([{"mu": [0.1, -0.05, 5.0], "scale": 1.2, "opacity": 0.5},
                   {"mu": [-0.2, 0.1, 5.5], "scale": 1.5, "opacity": 0.4},
                   {"mu": [0.05, 0.2, 6.0], "scale": 1.8, "opacity": 0.6}])
    v = synth.make_view(np.eye(3), np.zeros(3), 20.0, 20.0, 11.5, 9.5, 24, 20)
    return sc, v


@pytest.mark.parametrize("field", ["u", "v", "conic0", "conic1", "conic2", "opacity"])
def test_radiance_grad_geometry_finite_differences(orc, field):
    sc, v = _smooth_fixture()
    o = orc.render(sc, v)
    assert (o["flags"] == 0).all()
    rec, keys = o["rec"], o["keys"]
    rng = np.random.default_rng(7)
    gC = rng.standard_normal((3, 20, 24)).astype(np.float32)
    gD = rng.standard_normal((20, 24)).astype(np.float32)
    gA = rng.standard_normal((20, 24)).astype(np.float32)
    grad, _ = orc.radiance_backward(v, rec, keys, gC, gD, gA)
    for i in range(len(rec["gid"])):
        r2 = {k: np.array(a, copy=True) for k, a in rec.items() if isinstance(a, np.ndarray)}
        r3 = {k: np.array(a, copy=True) for k, a in rec.items() if isinstance(a, np.ndarray)}
        if field.startswith("conic"):
            c = int(field[-1])
            # conic ~0.03, p depends on it through dx^2 (<= 144 px^2): a small step keeps the
            # central difference's truncation error ~1e-3; the fp32 alpha noise is ~1e-5
            h = 1e-4
            r2["conic"][i, c] += h; r3["conic"][i, c] -= h
            # chain through e = k conic (e_b = 2k conic_b)
            an = grad[i, 2 + c] * float(K2) * (2.0 if c == 1 else 1.0)
        else:
            h = 1e-2
            r2[field][i] += h; r3[field][i] -= h
            an = grad[i, {"u": 0, "v": 1, "opacity": 5}[field]]
        fd = (_loss(orc, v, r2, keys, gC, gD, gA) - _loss(orc, v, r3, keys, gC, gD, gA)) / (2 * h)
        assert abs(fd - an) <= 5e-3 * max(abs(an), 1e-3), (i, fd, an)


# ------------------------------------------------------------------ projection backward (dL/dmu)
@pytest.mark.parametrize("axis", [0, 1, 2])
def test_mean_grad_finite_differences(orc, axis):
    """dL/dmu (oracle/backward.py chaining the record gradients through O1-O7)
    equals central differences of the whole pipeline (project -> bin -> composite)
    on the smooth fixture."""
    from oracle import backward as OB
    sc, v = _smooth_fixture()
    rng = np.random.default_rng(11)
    gC = rng.standard_normal((3, 20, 24)).astype(np.float32)
    gD = rng.standard_normal((20, 24)).astype(np.float32)
    gA = rng.standard_normal((20, 24)).astype(np.float32)
    P = orc.Params()

    def loss(scene):
        rec = orc.project(scene, v, P)
        keys = orc.bin_keys(rec, v)
        return orc.radiance_backward(v, rec, keys, gC, gD, gA, P)[1]

    rec = orc.project(sc, v, P)
    keys = orc.bin_keys(rec, v)
    grec, _ = orc.radiance_backward(v, rec, keys, gC, gD, gA, P)
    gmu = OB.mean_backward(sc, v, rec, grec, P)
    h = 1e-2
    for r, g in enumerate(rec["gid"]):
        s2, s3 = dataclasses.replace(sc, pos=sc.pos.copy()), dataclasses.replace(sc, pos=sc.pos.copy())
        s2.pos[axis, g] += h
        s3.pos[axis, g] -= h
        fd = (loss(s2) - loss(s3)) / (2 * h)
        assert abs(fd - gmu[r, axis]) <= 5e-3 * max(abs(gmu[r, axis]), 1e-2), (r, fd, gmu[r, axis])


def test_mean_grad_with_clamped_jacobian(orc):
    """A Gaussian far outside the frustum's x range (clamped J, reading Q6) whose
    footprint still reaches the image: the clamp branch of the chain."""
    from helpers import scene_of
    from oracle import backward as OB
    sc = scene_of([{"mu": [-6.0, 0.0, 5.0], "scale": 3.0, "opacity": 0.6}])
    v = synth.make_view(np.eye(3), np.zeros(3), 20.0, 20.0, 11.5, 9.5, 24, 20)
    P = orc.Params()
    rec = orc.project(sc, v, P)
    assert len(rec["gid"]) == 1
    xn = -6.0 / 5.0
    assert xn < (-(0.15 * 24) - 11.5) / 20.0               # clamped
    rng = np.random.default_rng(12)
    gC = rng.standard_normal((3, 20, 24)).astype(np.float32)
    z = np.zeros((20, 24), np.float32)

    def loss(scene):
        r = orc.project(scene, v, P)
        return orc.radiance_backward(v, r, orc.bin_keys(r, v), gC, z, z, P)[1]

    grec, _ = orc.radiance_backward(v, rec, orc.bin_keys(rec, v), gC, z, z, P)
    gmu = OB.mean_backward(sc, v, rec, grec, P)
    for axis in range(3):
        s2, s3 = dataclasses.replace(sc, pos=sc.pos.copy()), dataclasses.replace(sc, pos=sc.pos.copy())
        s2.pos[axis, 0] += 1e-2
        s3.pos[axis, 0] -= 1e-2
        fd = (loss(s2) - loss(s3)) / 2e-2
        assert abs(fd - gmu[0, axis]) <= 5e-3 * max(abs(gmu[0, axis]), 1e-2), (axis, fd, gmu[0, axis])


def test_sh_basis_gradient_equals_finite_differences_of_sh_color(orc):
    """backward.sh_basis_grad (numpy, term-by-term derivatives) against central
    differences of the C oracle's O10 colour (a separate implementation of the
    basis), for every degree, coefficient and axis (off the sphere: the basis
    polynomials are evaluated at the perturbed, unnormalised point)."""
    from oracle import backward as OB
    rng = np.random.default_rng(31)
    for deg in range(4):
        nk = (deg + 1) ** 2
        for _ in range(5):
            d = rng.standard_normal(3)
            d /= np.linalg.norm(d)
            coeff = rng.standard_normal((nk, 3))
            coeff[0] = 60.0                                 # keep every channel above the clamp
            an = OB.sh_basis_grad(deg, d).T @ coeff          # [3 axes][3 channels]
            for ax in range(3):
                e = np.zeros(3); e[ax] = 1e-6
                fd = (orc.sh_color(deg, coeff, d + e) - orc.sh_color(deg, coeff, d - e)) / 2e-6
                np.testing.assert_allclose(fd, an[ax], rtol=1e-6, atol=1e-7)


@pytest.mark.parametrize("axis", [0, 1, 2])
def test_mean_grad_finite_differences_with_view_dependent_colour(orc, axis):
    """The smooth fixture with degree-3 SH colour and a camera close enough that
    the view direction turns noticeably across a step: dL/dmu, including the SH
    direction term, equals central differences of the whole pipeline."""
    from helpers import scene_of
    from oracle import backward as OB
    rng = np.random.default_rng(41)
    gs = []
    for mu, s, o in (([0.1, -0.05, 2.0], 0.5, 0.5), ([-0.2, 0.1, 2.2], 0.6, 0.4), ([0.05, 0.2, 2.4], 0.7, 0.6)):
        sh = 0.3 * rng.standard_normal(48)
        sh[0:3] = 0.0                                       # base colour 0.5 keeps every channel > 0
        gs.append({"mu": mu, "scale": s, "opacity": o, "sh": sh})
    sc = scene_of(gs, sh_degree=3)
    v = synth.make_view(np.eye(3), np.zeros(3), 8.0, 8.0, 11.5, 9.5, 24, 20)
    P = orc.Params()
    gC = rng.standard_normal((3, 20, 24)).astype(np.float32)
    z = np.zeros((20, 24), np.float32)

    def loss(scene):
        r = orc.project(scene, v, P)
        return orc.radiance_backward(v, r, orc.bin_keys(r, v), gC, z, z, P)[1]

    rec = orc.project(sc, v, P)
    assert (rec["rgb"] > 0).all()
    o = orc.render(sc, v)
    assert (o["flags"] == 0).all()
    grec, _ = orc.radiance_backward(v, rec, orc.bin_keys(rec, v), gC, z, z, P)
    gmu = OB.mean_backward(sc, v, rec, grec, P)
    # the same chain with the colour's direction dependence dropped
    gmu0 = OB.mean_backward(dataclasses.replace(sc, sh_degree=0, sh=sc.sh[:3].copy()), v, rec, grec, P)
    assert np.abs(gmu - gmu0).max() > 1e-2 * np.abs(gmu).max()   # the SH term matters here
    h = 1e-3
    for r, g in enumerate(rec["gid"]):
        s2, s3 = dataclasses.replace(sc, pos=sc.pos.copy()), dataclasses.replace(sc, pos=sc.pos.copy())
        s2.pos[axis, g] += h
        s3.pos[axis, g] -= h
        fd = (loss(s2) - loss(s3)) / (2 * h)
        assert abs(fd - gmu[r, axis]) <= 5e-3 * max(abs(gmu[r, axis]), 1e-2), (r, fd, gmu[r, axis])


# ------------------------------------------------------------------ projection backward (other parameters)
def test_sh_basis_equals_the_c_oracle_colour(orc):
    """backward.sh_basis (numpy) against the C oracle's O10 colour (a separate
    implementation): with coefficients e_k + a large base term the colour is
    linear and c = sum_k b_k f_k + 0.5 channel by channel."""
    from oracle import backward as OB
    rng = np.random.default_rng(51)
    for deg in range(4):
        nk = (deg + 1) ** 2
        for _ in range(5):
            d = rng.standard_normal(3)
            d /= np.linalg.norm(d)
            coeff = rng.standard_normal((nk, 3))
            coeff[0] = 60.0
            want = OB.sh_basis(deg, d) @ coeff + 0.5
            np.testing.assert_allclose(orc.sh_color(deg, coeff, d), want, rtol=1e-12, atol=1e-12)


def _aniso_fixture(deg):
    from helpers import scene_of
    rng = np.random.default_rng(61)
    gs = []
    for mu, s, o in (([0.1, -0.05, 2.0], [0.6, 0.35, 0.25], 0.5), ([-0.2, 0.1, 2.2], [0.45, 0.7, 0.3], 0.4),
                     ([0.05, 0.2, 2.4], [0.8, 0.4, 0.5], 0.6)):
        q = rng.standard_normal(4)
        q = q / np.linalg.norm(q) * 1.3                    # un-normalised on purpose (O4 normalises)
        sh = 0.3 * rng.standard_normal((deg + 1) ** 2 * 3)
        sh[0:3] = 0.0
        gs.append({"mu": mu, "scale": s, "opacity": o, "quat": q, "sh": sh})
    return scene_of(gs, sh_degree=deg)


@pytest.mark.parametrize("field", ["scale", "quat", "opacity", "sh"])
def test_param_grads_finite_differences(orc, field):
    """dL/d{scale, quat, opacity, SH} (oracle/backward.param_backward chaining the
    record gradients through O4-O7 and O10) equal central differences of the
    whole pipeline (project -> bin -> composite) on anisotropic, rotated
    Gaussians with degree-3 colour."""
    from oracle import backward as OB
    sc = _aniso_fixture(3)
    v = synth.make_view(np.eye(3), np.zeros(3), 8.0, 8.0, 11.5, 9.5, 24, 20)
    P = orc.Params()
    rng = np.random.default_rng(71)
    gC = rng.standard_normal((3, 20, 24)).astype(np.float32)
    gD = rng.standard_normal((20, 24)).astype(np.float32)
    gA = rng.standard_normal((20, 24)).astype(np.float32)

    def loss(scene):
        r = orc.project(scene, v, P)
        return orc.radiance_backward(v, r, orc.bin_keys(r, v), gC, gD, gA, P)[1]

    rec = orc.project(sc, v, P)
    assert (orc.render(sc, v)["flags"] == 0).all()
    grec, _ = orc.radiance_backward(v, rec, orc.bin_keys(rec, v), gC, gD, gA, P)
    got = OB.param_backward(sc, v, rec, grec, P)[field]
    arr = {"scale": sc.scale, "quat": sc.quat, "opacity": sc.opacity[None, :], "sh": sc.sh}[field]
    # a step can straddle a pixel's alpha >= 1/255 or stop threshold (the loss is only piecewise
    # smooth); a correct derivative matches the central difference at one of three steps
    hs = {"sh": (1e-2, 3e-3, 1e-3)}.get(field, (1e-3, 3e-4, 1e-4))
    checked = 0
    for r, g in enumerate(rec["gid"]):
        for i in range(arr.shape[0]):
            an = got[r] if field == "opacity" else got[r, i]
            fds = []
            for h in hs:
                s2 = dataclasses.replace(sc, **{k: getattr(sc, k).copy() for k in ("scale", "quat", "opacity", "sh")})
                s3 = dataclasses.replace(sc, **{k: getattr(sc, k).copy() for k in ("scale", "quat", "opacity", "sh")})
                a2 = {"scale": s2.scale, "quat": s2.quat, "opacity": s2.opacity[None, :], "sh": s2.sh}[field]
                a3 = {"scale": s3.scale, "quat": s3.quat, "opacity": s3.opacity[None, :], "sh": s3.sh}[field]
                a2[i, g] += h
                a3[i, g] -= h
                fds.append((loss(s2) - loss(s3)) / (2 * h))
            assert min(abs(fd - an) for fd in fds) <= 5e-3 * max(abs(an), 1e-2), (r, i, fds, an)
            checked += abs(an) > 1e-2
    assert checked > 0


# ------------------------------------------------------------------ Eq. 1 joint step: L_f through the geometry
def _smooth_feature_fixture():
    from helpers import scene_of
    rng = np.random.default_rng(31)
    feat = rng.standard_normal((3, 8)).astype(np.float32)
    sc = scene_of([{"mu": [0.1, -0.05, 5.0], "scale": 1.2, "opacity": 0.5},
                   {"mu": [-0.2, 0.1, 5.5], "scale": 1.5, "opacity": 0.4},
                   {"mu": [0.05, 0.2, 6.0], "scale": 1.8, "opacity": 0.6}], feat=feat)
    v = synth.make_view(np.eye(3), np.zeros(3), 20.0, 20.0, 11.5, 9.5, 24, 20)
    return sc, v


@pytest.mark.parametrize("field", ["u", "v", "conic0", "conic1", "conic2", "opacity"])
def test_feature_loss_geometry_gradient_finite_differences(orc, field):
    """Eq. 1-2: the feature term's gradient through the blend weights
    into each record's (u, v, conic, opacity) -- central differences of
    L = sum_px gF(px) . F(px) (the forward composite) on the smooth fixture."""
    sc, v = _smooth_feature_fixture()
    o = orc.render(sc, v)
    assert (o["flags"] == 0).all()
    rec, keys = o["rec"], o["keys"]
    rng = np.random.default_rng(8)
    z3 = np.zeros((3, 20, 24), np.float32)
    z1 = np.zeros((20, 24), np.float32)
    gF = rng.standard_normal((8, 20, 24)).astype(np.float32)
    grad, loss = orc.radiance_backward(v, rec, keys, z3, z1, z1, feat=sc.feat, gF=gF)
    np.testing.assert_allclose(loss, float((gF.astype(np.float64) * o["feat"]).sum()), rtol=1e-6)
    lossf = lambda r: orc.radiance_backward(v, r, keys, z3, z1, z1, feat=sc.feat, gF=gF)[1]
    for i in range(len(rec["gid"])):
        r2 = {k: np.array(a, copy=True) for k, a in rec.items() if isinstance(a, np.ndarray)}
        r3 = {k: np.array(a, copy=True) for k, a in rec.items() if isinstance(a, np.ndarray)}
        if field.startswith("conic"):
            c = int(field[-1])
            h = 1e-4
            r2["conic"][i, c] += h; r3["conic"][i, c] -= h
            an = grad[i, 2 + c] * float(K2) * (2.0 if c == 1 else 1.0)
        else:
            h = 1e-2
            r2[field][i] += h; r3[field][i] -= h
            an = grad[i, {"u": 0, "v": 1, "opacity": 5}[field]]
        fd = (lossf(r2) - lossf(r3)) / (2 * h)
        assert abs(fd - an) <= 5e-3 * max(abs(an), 1e-3), (i, fd, an)
    assert np.abs(grad[:, 6:]).max() == 0          # the feature term moves no colour / depth


def test_feature_term_adds_linearly(orc):
    """grad(gC, gD, gA, gF) = grad(gC, gD, gA) + grad(0, 0, 0, gF) (the loss is linear
    in the upstream gradients) on a random tiny scene with features."""
    rng = np.random.default_rng(90)
    sc = random_tiny_scene(rng, 150, feat_dim=8, sh_degree=1)
    v = synth.make_view(np.eye(3), np.zeros(3), 40.0, 40.0, 23.5, 17.5, 48, 36)
    o = orc.render(sc, v)
    gC = rng.standard_normal((3, 36, 48)).astype(np.float32)
    gD = rng.standard_normal((36, 48)).astype(np.float32)
    gA = rng.standard_normal((36, 48)).astype(np.float32)
    gF = rng.standard_normal((8, 36, 48)).astype(np.float32)
    a, la = orc.radiance_backward(v, o["rec"], o["keys"], gC, gD, gA)
    b, lb = orc.radiance_backward(v, o["rec"], o["keys"], 0 * gC, 0 * gD, 0 * gA, feat=sc.feat, gF=gF)
    c, lc = orc.radiance_backward(v, o["rec"], o["keys"], gC, gD, gA, feat=sc.feat, gF=gF)
    np.testing.assert_allclose(c, a + b, rtol=1e-9, atol=1e-9)
    np.testing.assert_allclose(lc, la + lb, rtol=1e-9)
    assert np.abs(b[:, :6]).max() > 0
