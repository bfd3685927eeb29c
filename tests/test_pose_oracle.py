"""Pins of the oracle's N2 pose stage (Eq. 10) and of
Algorithm 2: forward-projection and
outlier-injection fixtures, degenerate input, noise
monotonicity, finite-difference Jacobian, and the Alg. 2 examples."""
import math

import numpy as np
import pytest

from oracle import pose as OP


def _rot(axis, deg):
    a = np.asarray(axis, np.float64)
    return OP.so3_exp(a / np.linalg.norm(a) * math.radians(deg))


def _scene(rng, n, extent=100.0):
    """A nadir-ish camera 150 m above points spread over the ground."""
    R = _rot([1, 0, 0], 180.0)                       # looking down
    C = np.array([0.0, 0.0, 150.0])
    t = -R @ C
    X = np.stack([rng.uniform(-extent / 2, extent / 2, n), rng.uniform(-extent / 2, extent / 2, n),
                  rng.uniform(0, 20, n)], 1)
    K = (800.0, 800.0, 511.5, 383.5)
    return K, R, t, X


def _project(K, R, t, X):
    Pc = X @ R.T + t
    return np.stack([K[0] * Pc[:, 0] / Pc[:, 2] + K[2], K[1] * Pc[:, 1] / Pc[:, 2] + K[3]], 1)


def _perturb(R, t, rng, deg=2.0, trans=1.0):
    dR = _rot(rng.standard_normal(3), deg)
    return dR @ R, t + rng.standard_normal(3) / math.sqrt(3) * trans


def _err(R, t, Rg, tg):
    """Rotation error in degrees from the chordal distance (well conditioned at 0,
    unlike arccos of the trace), translation distance."""
    c = np.linalg.norm(np.asarray(R) - np.asarray(Rg)) / (2.0 * math.sqrt(2.0))
    return math.degrees(2.0 * math.asin(min(1.0, c))), float(np.linalg.norm(np.asarray(t) - np.asarray(tg)))


def test_jacobian_matches_finite_differences():
    rng = np.random.default_rng(0)
    K, R, t, X = _scene(rng, 5)
    p2 = _project(K, R, t, X) + 3.0
    r0, _, Pc = OP.residuals(K, R, t, p2, X)
    J = OP.jacobian(K, Pc)
    eps = 1e-6
    for k in range(6):
        xi = np.zeros(6)
        xi[k] = eps
        R1, t1 = OP.apply(R, t, xi)
        r1, _, _ = OP.residuals(K, R1, t1, p2, X)
        np.testing.assert_allclose((r1 - r0) / eps, J[:, :, k], rtol=1e-4, atol=1e-4)


@pytest.mark.parametrize("seed", range(10))
def test_s418_noise_free_recovery(seed):
    """20 noise-free correspondences from a known pose -> within 1e-6 deg
    and 1e-6 * extent (from a start 2 deg / 1 m off, the dense-stage situation)."""
    rng = np.random.default_rng(seed)
    K, R, t, X = _scene(rng, 20)
    p2 = _project(K, R, t, X)
    R0, t0 = _perturb(R, t, rng)
    out = OP.solve_pnp(K, R0, t0, p2, X, tau=2.0, seed=seed)
    th, d = _err(out["R"], out["t"], R, t)
    assert th < 1e-6 and d < 1e-6 * 100.0, (th, d)
    assert out["n_inliers"] == 20 and out["mean_err"] < 1e-6


@pytest.mark.parametrize("seed", range(10))
def test_s419_outliers_rejected(seed):
    """+ 40% uniform-random outliers, tau = 2 px -> inliers = exactly the clean 20."""
    rng = np.random.default_rng(100 + seed)
    K, R, t, X = _scene(rng, 20)
    p2 = _project(K, R, t, X)
    n_out = 14                                   # 14 / 34 = 41 %
    Xo = np.stack([rng.uniform(-50, 50, n_out), rng.uniform(-50, 50, n_out), rng.uniform(0, 20, n_out)], 1)
    po = np.stack([rng.uniform(0, 1024, n_out), rng.uniform(0, 768, n_out)], 1)
    R0, t0 = _perturb(R, t, rng)
    out = OP.solve_pnp(K, R0, t0, np.concatenate([p2, po]), np.concatenate([X, Xo]), tau=2.0, seed=seed)
    assert out["inliers"][:20].all() and not out["inliers"][20:].any()
    th, d = _err(out["R"], out["t"], R, t)
    assert th < 1e-6 and d < 1e-4, (th, d)


def test_s420_degenerate_collinear_no_nan():
    rng = np.random.default_rng(5)
    K, R, t, _ = _scene(rng, 4)
    X = np.array([[0, 0, 0], [1, 1, 0], [2, 2, 0], [3, 3, 0]], np.float64)
    p2 = _project(K, R, t, X)
    out = OP.solve_pnp(K, R, t, p2, X, tau=2.0)
    assert np.isfinite(out["R"]).all() and np.isfinite(out["t"]).all()


def test_s423_noise_monotonicity():
    """Median pose error is non-decreasing in pixel noise sigma in {0, 0.5, 1}."""
    med = []
    for sigma in (0.0, 0.5, 1.0):
        errs = []
        for seed in range(12):
            rng = np.random.default_rng(200 + seed)
            K, R, t, X = _scene(rng, 40)
            p2 = _project(K, R, t, X) + sigma * rng.standard_normal((40, 2))
            R0, t0 = _perturb(R, t, rng)
            out = OP.solve_pnp(K, R0, t0, p2, X, tau=5.0, seed=seed)
            errs.append(_err(out["R"], out["t"], R, t)[0])
        med.append(float(np.median(errs)))
    assert med[0] <= med[1] <= med[2], med


def test_sample_index_distinct_and_in_range():
    for n in (3, 4, 17, 5000):
        for h in range(50):
            s = OP.minimal_sample(7, h, n)
            assert len(s) == 3 and len(set(s)) == 3 and all(0 <= i < n for i in s)


def test_alg2_examples():
    """identical poses -> reliable (0, 0); 25 deg apart -> unreliable;
    19.9 deg -> reliable.  Trace clamp keeps arccos finite for a rounding-perturbed R."""
    R, t = np.eye(3), np.zeros(3)
    assert OP.pose_difference(R, t, R, t) == (0.0, 0.0)
    assert OP.verify_consistency([(R, t)] * 3) == ("reliable", 2)
    R25 = _rot([0, 1, 0], 25.0)
    assert OP.verify_consistency([(R, t), (R, t), (R25, t)]) == ("unreliable", 1)
    R199 = _rot([0, 0, 1], 19.9)
    assert OP.verify_consistency([(R, t), (R199, t + 5.0)]) == ("reliable", 1)
    th, _ = OP.pose_difference(R * (1 + 1e-12), t, R, t)
    assert th == 0.0
    assert OP.verify_consistency([(R, t)]) == ("unreliable", -1)
