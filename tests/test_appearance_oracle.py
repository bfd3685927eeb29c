"""Pins of oracle/appearance.py (Eq. 3's L1 term against the appearance-varied
rendering I^a, reading Q38): the identity transform reduces to the plain L1 of
I^r; the loss is piecewise linear, so central differences away from its kinks
equal the gradient exactly (fp64); a uniform exposure change of the target is
fitted exactly by a = gain (zero loss)."""
import numpy as np

from oracle.appearance import appearance_l1


def _data(seed, P=6, H=9, W=11):
    rng = np.random.default_rng(seed)
    r = rng.uniform(0, 1, (P, H, W))
    t = rng.uniform(0, 1, (P, H, W))
    a = rng.uniform(0.7, 1.3, P)
    b = rng.uniform(-0.1, 0.1, P)
    return rng, r, t, a, b


def test_identity_transform_is_plain_l1():
    _, r, t, _, _ = _data(0)
    P = r.shape[0]
    loss, g_r, _, _ = appearance_l1(r, t, np.ones(P), np.zeros(P), 0.5)
    assert np.isclose(loss, 0.5 * np.abs(r - t).sum())
    np.testing.assert_array_equal(g_r, 0.5 * np.sign(r - t))


def test_central_differences_equal_the_gradient():
    rng, r, t, a, b = _data(1)
    loss, g_r, g_a, g_b = appearance_l1(r, t, a, b, 0.25)
    h = 1e-7
    margin = np.abs(a[:, None, None] * r + b[:, None, None] - t)
    for p in range(r.shape[0]):
        if margin[p].min() < 1e-4:
            continue
        a2, a3 = a.copy(), a.copy()
        a2[p] += h; a3[p] -= h
        fd = (appearance_l1(r, t, a2, b, 0.25)[0] - appearance_l1(r, t, a3, b, 0.25)[0]) / (2 * h)
        assert abs(fd - g_a[p]) <= 1e-6 * max(1.0, abs(g_a[p]))
        b2, b3 = b.copy(), b.copy()
        b2[p] += h; b3[p] -= h
        fd = (appearance_l1(r, t, a, b2, 0.25)[0] - appearance_l1(r, t, a, b3, 0.25)[0]) / (2 * h)
        assert abs(fd - g_b[p]) <= 1e-6 * max(1.0, abs(g_b[p]))
    for _ in range(20):
        p, y, x = (int(rng.integers(n)) for n in r.shape)
        if margin[p, y, x] < 1e-4:
            continue
        r2, r3 = r.copy(), r.copy()
        r2[p, y, x] += h; r3[p, y, x] -= h
        fd = (appearance_l1(r2, t, a, b, 0.25)[0] - appearance_l1(r3, t, a, b, 0.25)[0]) / (2 * h)
        assert abs(fd - g_r[p, y, x]) <= 1e-6


def test_exposure_change_is_fitted_exactly():
    _, r, _, _, _ = _data(2)
    gain = np.linspace(0.6, 1.4, r.shape[0])
    t = gain[:, None, None] * r
    loss, _, g_a, g_b = appearance_l1(r, t, gain, np.zeros(r.shape[0]), 1.0)
    assert loss < 1e-12
