"""Pins of the CPU oracle against things other than itself (task rule 3).

Every test names the passage / reading it pins.  Expected values come from
tests/golden/fixtures.json (SPEC.md examples + hand-derived closed forms),
textbook identities, independent library routines (scipy Rotation,
scipy.special.sph_harm_y, numpy.linalg.eigvalsh, finite differences) or
brute force.  No value here comes from the CUDA path.
"""
import math

import numpy as np
import pytest
from scipy.spatial.transform import Rotation
from scipy.special import sph_harm_y

import synth
from helpers import SH_C0, cam, golden, random_tiny_scene, scene_of

F32 = np.float32


def _one(orc, g, camera, **kw):
    sc = scene_of([g], **kw)
    return orc.project(sc, camera)


# ---------------------------------------------------------------- O1-O3, O2
def test_F1_principal_axis_projection(orc):
    """S:44 / Alg.1 l.9-12: (0,0,5) -> (50,50), depth 5."""
    fx = golden("F1")
    rec = _one(orc, {"mu": fx["mu"], "scale": 0.1}, cam(fx["camera"]))
    assert len(rec["gid"]) == 1
    assert rec["u"][0] == fx["expected"]["u"] and rec["v"][0] == fx["expected"]["v"]
    assert rec["z"][0] == fx["expected"]["z"]
    assert orc.tiles(cam(fx["camera"])) == tuple(fx["expected"]["tiles"])


def test_F1b_behind_camera_is_culled(orc):
    """(0,0,-5) is not in bounds -> near-culled and counted."""
    fx = golden("F1b")
    rec = _one(orc, {"mu": fx["mu"]}, cam(golden("F1")["camera"]))
    assert len(rec["gid"]) == 0 and rec["diag"]["near"] == 1


def test_cull_counters(orc):
    """O2 / S:158: degenerate, transparent, off-screen are skipped and counted."""
    c = cam(golden("F1")["camera"])
    sc = scene_of([{"mu": [0, 0, 5], "scale": [0.1, 0.0, 0.1]},           # zero scale -> degenerate
                   {"mu": [0, 0, 5], "opacity": 0.001},                    # < 1/255 -> transparent
                   {"mu": [-10.0, 0, 5], "scale": 0.01},                   # u = -150 -> off-screen
                   {"mu": [0, 0, 0.1]},                                    # z < z_near
                   {"mu": [0, 0, 5], "quat": [0, 0, 0, 0]},                # zero quaternion -> degenerate
                   {"mu": [0, 0, 5]}])
    rec = orc.project(sc, c)
    assert list(rec["gid"]) == [5]
    assert rec["diag"] == dict(near=1, transparent=1, degenerate=2, offscreen=1)


def test_projection_backprojection_round_trip(orc):
    """S:46 round trip (fp32 -> relative 1e-6): world points built in fp64 from
    chosen pixel centres and depths project onto those pixels, and O13 maps the
    depth there back onto the world point."""
    rng = np.random.default_rng(46)
    for _ in range(20):
        R = Rotation.random(random_state=rng).as_matrix()
        t = rng.uniform(-3, 3, 3)
        v = synth.make_view(R, t, 120.0, 110.0, 40.5, 30.5, 80, 60)
        Rf, tf = v.R.astype(np.float64), v.t.astype(np.float64)
        px, py, z = int(rng.integers(0, 80)), int(rng.integers(0, 60)), rng.uniform(1, 20)
        pc = np.array([(px - v.cx) / v.fx * z, (py - v.cy) / v.fy * z, z])
        X = Rf.T @ (pc - tf)
        rec = _one(orc, {"mu": X, "scale": 0.01}, v)
        assert len(rec["gid"]) == 1
        assert abs(rec["u"][0] - px) <= 2e-6 * max(1.0, abs(v.fx * pc[0] / z)) + 1e-4
        assert abs(rec["v"][0] - py) <= 2e-6 * max(1.0, abs(v.fy * pc[1] / z)) + 1e-4
        assert abs(rec["z"][0] - z) <= 1e-6 * z
        depth = np.zeros((60, 80), np.float32)
        alpha = np.zeros((60, 80), np.float32)
        depth[py, px] = z
        alpha[py, px] = 1.0
        xyz, valid, _ = orc.backproject(v, depth, alpha, 0.5)
        assert valid[py, px] == 1 and valid.sum() == 1
        scale = max(1.0, np.abs(X).max())
        np.testing.assert_allclose(xyz[:, py, px], X, atol=2e-6 * scale * z)


# ---------------------------------------------------------------- O4-O7
def test_F2_isotropic_footprint(orc):
    """F2 closed form: Sigma' = ((f s/z)^2 + 0.3) I, conic = I/4.3, r = 7, rect [2,3]^2."""
    fx = golden("F2")
    rec = _one(orc, {"mu": fx["mu"], "scale": fx["scale"], "opacity": fx["opacity"]}, cam(fx["camera"]))
    e = fx["expected"]
    np.testing.assert_allclose(rec["cov"][0], [e["cov_diag"], 0, e["cov_diag"]], rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose(rec["conic"][0], [e["conic_diag"], 0, e["conic_diag"]], rtol=1e-6, atol=1e-7)
    assert rec["radius"][0] == e["radius"]
    assert list(rec["rect"][0]) == e["rect"]
    keys = orc.bin_keys(rec, cam(fx["camera"]))
    assert len(keys["tile"]) == e["pairs"]


def test_F4_F5_radius(orc):
    """F4 (aerial scale) and F5 (minimum footprint 0.3 px^2 -> r = 2)."""
    for name in ("F4", "F5"):
        fx = golden(name)
        rec = _one(orc, {"mu": fx["mu"], "scale": fx["scale"]}, cam(fx["camera"]))
        assert rec["radius"][0] == fx["expected"]["radius"], name
        if "cov_diag" in fx["expected"]:
            np.testing.assert_allclose(rec["cov"][0, 0], fx["expected"]["cov_diag"], rtol=1e-6)


@pytest.mark.parametrize("seed", range(5))
def test_isotropic_covariance_independent_of_quaternion(orc, seed):
    """O4: for isotropic s, Sigma = s^2 I for every q (q is normalised first, Q2):
    an un-normalised random q must give the on-axis closed form."""
    rng = np.random.default_rng(seed)
    q = rng.standard_normal(4) * rng.uniform(0.2, 5.0)
    c = cam(golden("F2")["camera"])
    rec = _one(orc, {"mu": [0, 0, 5], "scale": 0.1, "quat": q}, c)
    np.testing.assert_allclose(rec["cov"][0], [4.3, 0, 4.3], rtol=2e-6, atol=2e-6)


@pytest.mark.parametrize("theta_deg", [0.0, 30.0, 90.0, 135.0])
def test_anisotropic_axis_assignment(orc, theta_deg):
    """O4: q = (cos th/2, 0, 0, sin th/2) rotates x toward y (textbook);
    on-axis Sigma' = (f/z)^2 Rz diag(s0^2, s1^2) Rz^T + 0.3 I."""
    th = math.radians(theta_deg)
    s0, s1 = 0.2, 0.05
    c = cam(golden("F2")["camera"])
    rec = _one(orc, {"mu": [0, 0, 5], "scale": [s0, s1, 0.01],
                     "quat": [math.cos(th / 2), 0, 0, math.sin(th / 2)]}, c)
    k = (100.0 / 5.0) ** 2
    a = k * (s0 ** 2 * math.cos(th) ** 2 + s1 ** 2 * math.sin(th) ** 2) + 0.3
    b = k * (s0 ** 2 - s1 ** 2) * math.sin(th) * math.cos(th)
    cc = k * (s0 ** 2 * math.sin(th) ** 2 + s1 ** 2 * math.cos(th) ** 2) + 0.3
    np.testing.assert_allclose(rec["cov"][0], [a, b, cc], rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("seed", range(10))
def test_ewa_matches_finite_difference_jacobian(orc, seed):
    """O5 (textbook EWA, [3DGS] cited by P:132): for an on-screen mean,
    Sigma' = J Sigma_cam J^T + 0.3 I with J the Jacobian of the pinhole map at
    the mean -- here taken by central finite differences in fp64, and
    Sigma_world = R(q) diag(s^2) R(q)^T from scipy's Rotation (library)."""
    rng = np.random.default_rng(100 + seed)
    R = Rotation.random(random_state=rng).as_matrix()
    t = rng.uniform(-1, 1, 3)
    v = synth.make_view(R, t, 300.0, 280.0, 160.0, 120.0, 320, 240)
    Rf, tf = v.R.astype(np.float64), v.t.astype(np.float64)
    pc = np.array([rng.uniform(-0.3, 0.3) * 6, rng.uniform(-0.3, 0.3) * 6, 6.0])
    X = (Rf.T @ (pc - tf)).astype(np.float32)
    q = rng.standard_normal(4)
    q /= np.linalg.norm(q)
    s = np.exp(rng.uniform(math.log(0.02), math.log(0.3), 3))
    rec = _one(orc, {"mu": X, "scale": s, "quat": q}, v)
    assert len(rec["gid"]) == 1
    Rq = Rotation.from_quat([q[1], q[2], q[3], q[0]]).as_matrix()     # scipy order x,y,z,w
    Sw = Rq @ np.diag(s.astype(np.float32).astype(np.float64) ** 2) @ Rq.T
    Sc = Rf @ Sw @ Rf.T
    pcam = Rf @ X.astype(np.float64) + tf

    def pix(p):
        return np.array([v.fx * p[0] / p[2] + v.cx, v.fy * p[1] / p[2] + v.cy])

    h = 1e-5
    J = np.stack([(pix(pcam + h * e) - pix(pcam - h * e)) / (2 * h) for e in np.eye(3)], axis=1)
    S2 = J @ Sc @ J.T + 0.3 * np.eye(2)
    got = rec["cov"][0].astype(np.float64)
    scale = abs(S2).max()
    np.testing.assert_allclose(got, [S2[0, 0], S2[0, 1], S2[1, 1]], atol=2e-5 * scale)
    # O6: conic is the inverse
    a, b, c = got
    ca, cb, cc = rec["conic"][0].astype(np.float64)
    np.testing.assert_allclose(np.array([[ca, cb], [cb, cc]]) @ np.array([[a, b], [b, c]]), np.eye(2), atol=1e-5)
    # O7: r = ceil(3 sqrt(lambda_max)) with lambda_max from LAPACK (numpy eigvalsh)
    lam = np.linalg.eigvalsh(np.array([[a, b], [b, c]]))[-1]
    r_ref = 3.0 * math.sqrt(lam)
    if abs(r_ref - round(r_ref)) > 1e-4:
        assert rec["radius"][0] == math.ceil(r_ref)


def test_offscreen_jacobian_clamp(orc):
    """Q6 (parity unpinned convention, [3DGS] 1.3 tan(fov/2) guard): beyond
    0.15 W of the border the Jacobian stops growing, so the footprint of an
    isotropic Gaussian far off to the side equals that at the clamp."""
    c = cam(golden("F2")["camera"])
    lim = (1.15 * 100 - 50) / 100.0  # x/z at the clamp
    r1 = _one(orc, {"mu": [lim * 5 + 0.5, 0, 5], "scale": 0.5}, c)["cov"]
    r2 = _one(orc, {"mu": [lim * 5 + 1.0, 0, 5], "scale": 0.5}, c)["cov"]
    if len(r1) and len(r2):
        np.testing.assert_allclose(r1[0], r2[0], rtol=1e-6)


# ---------------------------------------------------------------- O8
def test_tile_rectangle_brute_force(orc):
    """O8 / Q10: the rectangle is exactly the set of tiles k whose half-open
    pixel interval [16k, 16k+16) meets [u - r, u + r], clamped to the grid."""
    rng = np.random.default_rng(8)
    v = synth.make_view(np.eye(3), np.zeros(3), 100.0, 100.0, 50.0, 40.0, 100, 80)
    n = 400
    sc = random_tiny_scene(rng, n)
    sc.pos[2] = np.abs(sc.pos[2]) + 1.0
    rec = orc.project(sc, v)
    TX, TY = orc.tiles(v)
    for i in range(len(rec["gid"])):
        u, vv, r = float(rec["u"][i]), float(rec["v"][i]), float(rec["radius"][i])
        kx = [k for k in range(TX) if (u - r) < 16 * k + 16 and (u + r) >= 16 * k]
        ky = [k for k in range(TY) if (vv - r) < 16 * k + 16 and (vv + r) >= 16 * k]
        x0, x1, y0, y1 = rec["rect"][i]
        assert kx == list(range(x0, x1 + 1)) and ky == list(range(y0, y1 + 1))
    # every off-screen cull really touches no tile
    assert rec["diag"]["offscreen"] >= 0


def test_F6_inclusive_upper_tile(orc):
    fx = golden("F6")
    rec = _one(orc, {"mu": fx["mu"], "scale": fx["scale"]}, cam(fx["camera"]))
    assert rec["u"][0] == fx["expected"]["u"] and rec["radius"][0] == fx["expected"]["radius"]
    assert [rec["rect"][0][0], rec["rect"][0][1]] == fx["expected"]["rect_x"]


# ---------------------------------------------------------------- O10 SH
def test_sh_degree0_identity(orc):
    """degree 0: rgb = Y_00 k0 + 0.5 with Y_00 = 1/(2 sqrt(pi)) (textbook)."""
    for k0 in (-1.0, 0.0, 0.37, 2.0):
        got = orc.sh_color(0, [[k0, 2 * k0, -k0]], [0, 0, 1])
        exp = np.maximum(np.array([k0, 2 * k0, -k0]) * SH_C0 + 0.5, 0)
        np.testing.assert_allclose(got, exp, rtol=1e-15, atol=1e-15)


def _fib_sphere(n):
    i = np.arange(n) + 0.5
    ph = math.pi * (3 - math.sqrt(5)) * i
    z = 1 - 2 * i / n
    r = np.sqrt(1 - z * z)
    return np.stack([r * np.cos(ph), r * np.sin(ph), z], axis=1)


def _basis_via_oracle(orc, deg, dirs):
    nk = (deg + 1) ** 2
    B = np.zeros((len(dirs), nk))
    big = 10.0 / SH_C0            # keep rgb > 0 so the clamp never acts
    for k in range(nk):
        coeff = np.zeros((nk, 3))
        coeff[0, :] = big
        coeff[k, 0] += 1.0
        for j, d in enumerate(dirs):
            # rgb_0 = sum_k' basis_k'(d) coeff_k' + 0.5 = 10 + basis_k(d) + 0.5
            B[j, k] = orc.sh_color(deg, coeff, d)[0] - 10.5
    return B


def test_sh_orthonormal_and_matches_scipy(orc):
    """O10: the 16 real SH basis functions are orthonormal on the sphere
    (quadrature), and |basis| equals |real Y_lm| from scipy.special.sph_harm_y
    in the m = -l..l order; signs are a convention (parity unpinned)."""
    dirs = _fib_sphere(3000)
    B = _basis_via_oracle(orc, 3, dirs)
    G = B.T @ B * (4 * math.pi / len(dirs))
    np.testing.assert_allclose(G, np.eye(16), atol=2e-3)
    theta = np.arccos(np.clip(dirs[:, 2], -1, 1))
    phi = np.arctan2(dirs[:, 1], dirs[:, 0])
    k = 0
    for l in range(4):
        for m in range(-l, l + 1):
            Y = sph_harm_y(l, abs(m), theta, phi)
            if m < 0:
                ref = math.sqrt(2) * (-1) ** m * Y.imag
            elif m == 0:
                ref = Y.real
            else:
                ref = math.sqrt(2) * (-1) ** m * Y.real
            np.testing.assert_allclose(np.abs(B[:, k]), np.abs(ref), atol=1e-9, err_msg=f"l={l} m={m}")
            k += 1


def test_sh_view_direction(orc):
    """O10: the colour is evaluated at d = (mu - c_cam)/|mu - c_cam| with
    c_cam = -R^T t: a degree-1 coefficient on the z-basis gives +C1 for a camera
    below the Gaussian looking up and -C1 for one above looking down."""
    coeff1 = np.zeros(12, np.float32)
    coeff1[0:3] = 1.0 / SH_C0   # rgb = 1.5 + b(d) > 0
    coeff1[6] = 1.0             # k=2 (z basis), channel 0
    g = {"mu": [0.0, 0.0, 0.0], "scale": 0.01, "sh": coeff1}
    sc = scene_of([g], sh_degree=1)
    up = synth.make_view(*synth.look_from([0, 0, -5], [0, 0, 1]), 100, 100, 50, 50, 100, 100)
    down = synth.make_view(*synth.look_from([0, 0, 5], [0, 0, -1]), 100, 100, 50, 50, 100, 100)
    c1 = math.sqrt(3.0 / (4.0 * math.pi))
    r_up = orc.project(sc, up)["rgb"][0, 0]
    r_dn = orc.project(sc, down)["rgb"][0, 0]
    np.testing.assert_allclose(r_up - 1.5, c1, rtol=1e-6)
    np.testing.assert_allclose(r_dn - 1.5, -c1, rtol=1e-6)


# ---------------------------------------------------------------- O11
def test_keys_sorted_counts_and_lower_bound_ranges(orc):
    """O11 / Q12 / Q13: keys lexicographic in (tile, depth_bits, gid); the sum
    of rectangle areas is P; ranges are lower bounds (empty tiles get s = e)."""
    sc, vs = synth.make_config("C1")
    v = vs[0]
    rec = orc.project(sc, v)
    k = orc.bin_keys(rec, v)
    P = int(((rec["rect"][:, 1] - rec["rect"][:, 0] + 1) * (rec["rect"][:, 3] - rec["rect"][:, 2] + 1)).sum())
    assert len(k["tile"]) == P
    trip = list(zip(k["tile"].tolist(), k["depth"].tolist(), k["gid"].tolist()))
    assert trip == sorted(trip) and len(set(trip)) == P
    np.testing.assert_array_equal(k["depth"], rec["z"][k["rec"]].view(np.uint32))
    tiles = k["tile"].astype(np.int64)
    T = k["ranges"].shape[0]
    np.testing.assert_array_equal(k["ranges"][:, 0], np.searchsorted(tiles, np.arange(T), "left"))
    np.testing.assert_array_equal(k["ranges"][:, 1], np.searchsorted(tiles, np.arange(T), "right"))


# ---------------------------------------------------------------- O12
def _render_one(orc, gs, camera, feat=None):
    sc = scene_of(gs, feat=feat)
    return orc.render(sc, camera), sc


def test_F2_compositing_closed_form(orc):
    """F2 / S:161: peak at (cx,cy), alpha = 0.99, Dz = 4.95, A = 0.99; at
    (52,50): alpha = 0.99 exp(-2/4.3)."""
    fx = golden("F2")
    e = fx["expected"]
    r, _ = _render_one(orc, [{"mu": fx["mu"], "scale": fx["scale"], "opacity": fx["opacity"],
                              "rgb": fx["rgb"]}], cam(fx["camera"]))
    cy, cx = 50, 50
    assert np.unravel_index(np.argmax(r["alpha"]), r["alpha"].shape) == (cy, cx)
    np.testing.assert_allclose(r["alpha"][cy, cx], e["alpha_center"], rtol=1e-6)
    np.testing.assert_allclose(r["depth"][cy, cx], e["depth_center"], rtol=1e-6)
    np.testing.assert_allclose(r["depth"][cy, cx] / r["alpha"][cy, cx], 5.0, rtol=1e-6)  # S:161 within 1%
    np.testing.assert_allclose(r["rgb"][:, cy, cx], 0.99 * np.array(fx["rgb"]), rtol=1e-6, atol=1e-7)
    a52 = 0.99 * math.exp(e["pixel_52_50_power"])
    np.testing.assert_allclose(r["alpha"][50, 52], a52, rtol=1e-6)


def test_F3_opacity_one_occlusion(orc):
    """F3 / S:162 / Q15: the rear layer after an alpha=0.99 front is stopped."""
    fx = golden("F3")
    r, _ = _render_one(orc, [fx["front"], fx["rear"]], cam(fx["camera"]))
    rec = r["rec"]
    np.testing.assert_allclose(rec["cov"][1, 0], fx["expected"]["rear_cov_diag"], rtol=1e-6)
    assert rec["radius"][1] == fx["expected"]["rear_radius"]
    assert list(rec["rect"][1]) == fx["expected"]["rear_rect"]
    # each tile lists the front then the rear
    for t in range(r["keys"]["ranges"].shape[0]):
        s, e = r["keys"]["ranges"][t]
        if e > s:
            assert list(r["keys"]["gid"][s:e]) == [0, 1]
    np.testing.assert_allclose(r["rgb"][:, 50, 50], fx["expected"]["center_rgb"], atol=1e-6)
    np.testing.assert_allclose(r["alpha"][50, 50], fx["expected"]["center_alpha"], rtol=1e-6)
    assert r["rgb"][2, 50, 50] < 1e-7                      # rear colour (blue) absent


def test_F7_ambiguity_flag(orc):
    """F7 / Q20: four alpha=0.9 layers leave T one ulp above 1e-4 -> flagged."""
    fx = golden("F7")
    gs = [{"mu": [0, 0, d], "scale": fx["scale"], "opacity": fx["opacity"]} for d in fx["depths"]]
    r, _ = _render_one(orc, gs, cam(fx["camera"]))
    assert r["flags"][50, 50] & fx["expected"]["center_flag_bit"]


def test_F8_alpha_cutoff(orc):
    """F8 / Q14: o = 1, sigma'^2 = 4.3: pixels with o exp(power) >= 1/255
    (2^-10 away from the cut) get alpha exactly min(0.99, exp(power)); pixels below get 0."""
    fx = golden("F8")
    r, _ = _render_one(orc, [{"mu": fx["mu"], "scale": fx["scale"], "opacity": 1.0, "rgb": [1, 1, 1]}],
                       cam(fx["camera"]))
    cut = 1.0 / 255.0
    checked = 0
    for py in range(40, 61):
        for px in range(40, 61):
            d2 = (px - 50) ** 2 + (py - 50) ** 2
            a = math.exp(-0.5 * d2 / 4.3)
            if a >= cut * (1 + 2 ** -10):
                np.testing.assert_allclose(r["alpha"][py, px], min(0.99, a), rtol=1e-5)
                checked += 1
            elif a <= cut * (1 - 2 ** -10):
                assert r["alpha"][py, px] == 0.0 and r["rgb"][0, py, px] == 0.0
                checked += 1
    assert checked > 300
    assert r["alpha"][50, 56] > 0 and r["alpha"][50, 57] == 0      # 6 < 6.90 < 7


def test_empty_scene(orc):
    """empty scene -> all zeros."""
    sc = scene_of([])
    v = synth.box_view()
    r = orc.render(sc, v)
    assert not r["rgb"].any() and not r["alpha"].any() and not r["depth"].any()


@pytest.mark.parametrize("seed", range(6))
def test_weights_sum_to_alpha_and_transmittance_bounds(orc, seed):
    """with all features = 1 the feature plane is sum(w),
    which must equal A = 1 - T <= 1 (fp32 accumulation, 1e-5)."""
    rng = np.random.default_rng(300 + seed)
    sc = random_tiny_scene(rng, 60, feat_dim=4)
    sc.feat[:] = 1.0
    r = orc.render(sc, synth.box_view())
    for c in range(4):
        np.testing.assert_allclose(r["feat"][c], r["alpha"], atol=1e-5)
    assert (r["alpha"] >= 0).all() and (r["alpha"] <= 1.0).all()


def test_feature_linearity(orc):
    """render(a f1 + b f2) = a render(f1) + b render(f2) within 1e-6."""
    rng = np.random.default_rng(175)
    sc = random_tiny_scene(rng, 80, feat_dim=8)
    f1 = rng.standard_normal((80, 8)).astype(np.float32)
    f2 = rng.standard_normal((80, 8)).astype(np.float32)
    v = synth.box_view()
    rec = orc.project(sc, v)
    keys = orc.bin_keys(rec, v)
    a, b = 0.75, -1.25
    r1 = orc.composite(v, rec, keys, f1)["feat"]
    r2 = orc.composite(v, rec, keys, f2)["feat"]
    r12 = orc.composite(v, rec, keys, (a * f1 + b * f2).astype(np.float32))["feat"]
    np.testing.assert_allclose(r12, a * r1 + b * r2, atol=1e-6)


def test_brute_force_identical_on_C1_and_fixtures(orc):
    """Pin of O11+O12: the binned render equals, bit for bit, the per-pixel
    brute force over all Gaussians (C1 + SPEC fixtures)."""
    cases = [synth.make_config("C1")]
    for name in ("F2", "F3", "F8"):
        fx = golden(name)
        gs = [fx["front"], fx["rear"]] if name == "F3" else [{"mu": fx["mu"], "scale": fx["scale"],
                                                             "opacity": fx.get("opacity", 0.99)}]
        cases.append((scene_of(gs), [cam(fx["camera"])]))
    for sc, vs in cases:
        v = vs[0]
        r = orc.render(sc, v)
        bf = orc.brute_force(v, r["rec"], sc.feat)
        for k in ("rgb", "depth", "alpha", "flags"):
            np.testing.assert_array_equal(r[k], bf[k])


@pytest.mark.parametrize("seed", range(100))
def test_brute_force_identical_random_tiny(orc, seed):
    """100 random tiny scenes (5-50 Gaussians, depth ties, off-screen, behind
    camera, un-normalised q, features, SH 1): bit-identical to brute force."""
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(5, 51))
    sc = random_tiny_scene(rng, n, feat_dim=4 if seed % 2 else 0, sh_degree=seed % 2)
    v = synth.make_view(np.eye(3), np.zeros(3), 40.0, 44.0, 23.5, 17.0, 48, 36)
    r = orc.render(sc, v)
    bf = orc.brute_force(v, r["rec"], sc.feat)
    for k in ("rgb", "depth", "alpha", "feat", "flags"):
        np.testing.assert_array_equal(r[k], bf[k])


# ---------------------------------------------------------------- O13
def test_backproject_fronto_parallel_plane(orc):
    """O13: a fronto-parallel constant-z layer gives Dz/A = z at every covered
    pixel, so the back-projected points lie on the plane and re-project to
    their own pixels (S:46 round trip on rendered depth)."""
    rng = np.random.default_rng(13)
    gs = [{"mu": [float(x), float(y), 5.0], "scale": 0.12, "opacity": float(o)}
          for x, y, o in zip(rng.uniform(-2, 2, 1500), rng.uniform(-2, 2, 1500), rng.uniform(0.3, 1, 1500))]
    R = Rotation.from_euler("xyz", [0.0, 0.0, 0.3]).as_matrix()     # rotation about the optical axis keeps z
    v = synth.make_view(R, np.zeros(3), 64.0, 64.0, 31.5, 31.5, 64, 64)
    sc = scene_of([dict(g, mu=list(R.T @ np.array(g["mu"]))) for g in gs])
    r = orc.render(sc, v, a_min=0.5)
    m = r["valid"] > 0
    assert m.sum() > 500
    zbar = r["depth"][m].astype(np.float64) / r["alpha"][m]
    np.testing.assert_allclose(zbar, 5.0, rtol=2e-5)
    Rf = v.R.astype(np.float64)
    pc = np.einsum("ij,jhw->ihw", Rf, r["xyz"].astype(np.float64))
    np.testing.assert_allclose(pc[2][m], 5.0, rtol=2e-5)
    ys, xs = np.nonzero(m)
    np.testing.assert_allclose(v.fx * pc[0][m] / pc[2][m] + v.cx, xs, atol=1e-3)
    np.testing.assert_allclose(v.fy * pc[1][m] / pc[2][m] + v.cy, ys, atol=1e-3)
    assert not r["xyz"][:, ~m].any()


def test_defaults_match_readings(orc):
    """Q5, Q6, Q7, Q14, Q15 defaults."""
    p = orc.Params()
    assert (p.z_near, p.dilation, p.clamp_margin, p.alpha_max, p.t_min) == (0.2, 0.3, 0.15, 0.99, 1e-4)
    assert p.alpha_min == 1.0 / 255.0
