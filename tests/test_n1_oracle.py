"""Pins of the oracle's N1 row: Alg. 1 render visibility with
projection filtering (forward criterion of SPEC S:180) and
significance scoring Eq. 4-6.  Fixtures follow SPEC S:169-171
(visibility examples) and S:281-282 (scoring examples); invariants: the sum
of all contributions equals the sum of rendered opacity, and the per-record
contributions of the binned render equal those of the per-pixel brute force."""
import math

import numpy as np
import pytest

import synth
from helpers import cam, golden, random_tiny_scene, scene_of


def _cam100():
    return cam(golden("F1")["camera"])


def _vis(orc, sc, v, feat=None, fmap=None, stride=1, eps=1e-6):
    r = orc.render(sc, v)
    vis, ssum, cnt = orc.visibility_score(v, r["rec"], r["contrib"], sc.n, eps, feat, fmap, stride)
    return r, vis, ssum, cnt


def test_s169_on_axis_gaussian_visible_at_principal_point(orc):
    """one Gaussian on the principal axis, no occluders -> visible at (cx, cy)."""
    v = _cam100()
    sc = scene_of([{"mu": [0, 0, 5], "scale": 0.1, "opacity": 0.9}])
    r, vis, _, cnt = _vis(orc, sc, v)
    assert vis.tolist() == [1] and cnt.tolist() == [1]
    assert (r["rec"]["u"][0], r["rec"]["v"][0]) == (50.0, 50.0)


def test_s170_occluded_rear_not_visible(orc):
    """a small Gaussian behind a large opaque one is reached only after
    the transmittance cut-off -> zero contribution -> not visible."""
    v = _cam100()
    sc = scene_of([{"mu": [0, 0, 5], "scale": 1.0, "opacity": 1.0},      # covers the rear footprint at alpha 0.99
                   {"mu": [0, 0, 5.5], "scale": 1.0, "opacity": 1.0},
                   {"mu": [0, 0, 10], "scale": 0.05, "opacity": 1.0}])
    r, vis, _, cnt = _vis(orc, sc, v)
    assert r["contrib"][2] == 0.0
    assert vis.tolist() == [1, 1, 0]


def test_s171_offscreen_centre_excluded_by_bounds(orc):
    """a Gaussian projecting to u = -10 is excluded by M^i even though
    its footprint contributes to on-screen pixels."""
    v = _cam100()
    x = (-10 - 50) * 5 / 100.0          # u = 100 * x / 5 + 50 = -10
    sc = scene_of([{"mu": [x, 0, 5], "scale": 0.8, "opacity": 0.9}])
    r, vis, _, cnt = _vis(orc, sc, v)
    assert abs(r["rec"]["u"][0] + 10.0) < 1e-4
    assert r["contrib"][0] > 1.0            # it does blend into the image
    assert vis.tolist() == [0] and cnt.tolist() == [0]


def test_contributions_sum_to_total_opacity(orc):
    """Sum over Gaussians of sum over pixels of w = sum over pixels of A
    (sum_i w_i = accum_alpha per pixel)."""
    sc, vs = synth.make_config("C1")
    r = orc.render(sc, vs[0])
    np.testing.assert_allclose(r["contrib"].sum(), r["alpha"].astype(np.float64).sum(), rtol=1e-6)
    assert (r["contrib"] >= 0).all()


@pytest.mark.parametrize("seed", range(20))
def test_contributions_match_brute_force(orc, seed):
    """visibility agrees with a brute-force per-pixel contribution scan
    (<= 50 Gaussians): per-record sums are bit-identical."""
    rng = np.random.default_rng(700 + seed)
    sc = random_tiny_scene(rng, int(rng.integers(5, 51)))
    v = synth.make_view(np.eye(3), np.zeros(3), 40.0, 44.0, 23.5, 17.0, 48, 36)
    r = orc.render(sc, v)
    bf = orc.brute_force(v, r["rec"])
    np.testing.assert_array_equal(r["contrib"], bf["contrib"])


def test_s281_identical_features_score_one(orc):
    """feature equal to the sampled image feature, seen in 1 view -> 1.0."""
    v = _cam100()
    f = np.array([[0.3, -0.2, 0.9, 0.1]], np.float32)
    sc = scene_of([{"mu": [0, 0, 5], "scale": 0.1, "opacity": 0.9}], feat=f)
    fmap = np.zeros((4, 100, 100), np.float32)
    fmap[:, 50, 50] = 2.5 * f[0]                       # cosine is scale invariant
    _, vis, ssum, cnt = _vis(orc, sc, v, feat=f, fmap=fmap)
    np.testing.assert_allclose(orc.final_scores(ssum, cnt), [1.0], rtol=1e-12)


def test_s282_two_views_average(orc):
    """S:282 / Eq. 6: per-view scores 0.8 and 0.6 -> final 0.7 (S(g) = S(G)/M)."""
    v = _cam100()
    f = np.array([[1.0, 0.0]], np.float32)
    sc = scene_of([{"mu": [0, 0, 5], "scale": 0.1, "opacity": 0.9}], feat=f)
    ssum, cnt = np.zeros(1), np.zeros(1, np.int64)
    for c in (0.8, 0.6):
        fmap = np.zeros((2, 100, 100), np.float32)
        fmap[:, 50, 50] = [c, math.sqrt(1 - c * c)]
        r = orc.render(sc, v)
        orc.visibility_score(v, r["rec"], r["contrib"], 1, 1e-6, f, fmap, 1, ssum, cnt)
    np.testing.assert_allclose(orc.final_scores(ssum, cnt), [0.7], rtol=1e-6)
    assert cnt.tolist() == [2]


def test_unseen_gaussian_scores_minus_inf(orc):
    """final score is -inf when M = 0."""
    out = orc.final_scores(np.array([0.5, 0.0]), np.array([1, 0]))
    assert out[0] == 0.5 and out[1] == -np.inf


@pytest.mark.parametrize("stride,u,expect", [(1, 50.0, 50), (1, 50.45, 50), (1, 50.6, 51), (4, 50.0, 12),
                                             (4, 47.3, 11), (4, 47.7, 12), (8, 99.4, 12)])
def test_nearest_cell_sampling(orc, stride, u, expect):
    """Reading Q27: the target map is sampled at cell floor((u + 0.5)/stride)
    (pixel-centre convention, SPEC S:283 nearest-cell lookup)."""
    v = _cam100()
    f = np.array([[1.0, 0.0]], np.float32)
    x = (u - 50.0) * 5 / 100.0
    sc = scene_of([{"mu": [x, 0, 5], "scale": 0.1, "opacity": 0.9}], feat=f)
    r = orc.render(sc, v)
    uu = float(r["rec"]["u"][0])
    assert abs(uu - u) < 1e-4
    Wf = (100 + stride - 1) // stride
    fmap = np.zeros((2, Wf, Wf), np.float32)
    fmap[1] = 1.0                                        # orthogonal everywhere ...
    cell = int(math.floor((uu + 0.5) / stride))
    cy = int(math.floor((50.0 + 0.5) / stride))
    fmap[:, cy, cell] = [1.0, 0.0]                       # ... except at the expected cell
    assert cell == expect
    vis, ssum, cnt = orc.visibility_score(v, r["rec"], r["contrib"], 1, 1e-6, f, fmap, stride)
    assert ssum[0] == 1.0 and cnt[0] == 1
