"""Pins of oracle/ssim.py (Eq. 3's D-SSIM, reading Q37) against a brute-force
double loop over the window (no scipy) and the identities SSIM(x, x) = 1 and
symmetry."""
import numpy as np

from oracle import ssim as OS


def _brute(x, y):
    w = OS.window()
    C, H, W = x.shape
    S = np.zeros((C, H, W))
    for c in range(C):
        for i in range(H):
            for j in range(W):
                st = np.zeros(5)
                for di in range(-5, 6):
                    for dj in range(-5, 6):
                        ii, jj = i + di, j + dj
                        if 0 <= ii < H and 0 <= jj < W:
                            a, b, k = x[c, ii, jj], y[c, ii, jj], w[di + 5, dj + 5]
                            st += k * np.array([a, b, a * a, b * b, a * b])
                mx, my = st[0], st[1]
                sxx, syy, sxy = st[2] - mx * mx, st[3] - my * my, st[4] - mx * my
                S[c, i, j] = ((2 * mx * my + OS.C1) * (2 * sxy + OS.C2)) / \
                    ((mx * mx + my * my + OS.C1) * (sxx + syy + OS.C2))
    return S


def test_window_is_a_normalised_gaussian():
    w = OS.window()
    assert w.shape == (11, 11) and abs(w.sum() - 1.0) < 1e-15
    assert np.allclose(w, w.T) and w[5, 5] == w.max()
    assert abs(w[5, 6] / w[5, 5] - np.exp(-1 / (2 * 1.5 ** 2))) < 1e-12


def test_ssim_map_equals_brute_force():
    rng = np.random.default_rng(3)
    x = rng.uniform(0, 1, (2, 9, 13))
    y = np.clip(x + rng.normal(0, 0.2, x.shape), 0, 1)
    np.testing.assert_allclose(OS.ssim_map(x, y), _brute(x, y), rtol=1e-12, atol=1e-12)


def test_identities():
    rng = np.random.default_rng(4)
    x = rng.uniform(0, 1, (3, 16, 12))
    y = rng.uniform(0, 1, (3, 16, 12))
    assert abs(OS.dssim(x, x)) < 1e-12
    assert abs(OS.dssim(x, y) - OS.dssim(y, x)) < 1e-12
    assert 0.0 < OS.dssim(x, y) < 2.0


def test_dssim_grad_matches_central_differences():
    """The chain-rule gradient against fp64 central differences of dssim() at every
    pixel of a small ragged image (window overhangs every border)."""
    rng = np.random.default_rng(5)
    x = rng.uniform(0, 1, (2, 7, 12))
    y = np.clip(x + rng.normal(0, 0.15, x.shape), 0, 1)
    g = OS.dssim_grad(x, y)
    h = 1e-6
    fd = np.empty_like(x)
    for idx in np.ndindex(x.shape):
        xp, xm = x.copy(), x.copy()
        xp[idx] += h
        xm[idx] -= h
        fd[idx] = (OS.dssim(xp, y) - OS.dssim(xm, y)) / (2 * h)
    np.testing.assert_allclose(g, fd, rtol=1e-5, atol=1e-9)


def test_dssim_grad_vanishes_at_the_minimum():
    """x = y is the minimum of 1 - SSIM (S <= 1): the gradient is zero there."""
    rng = np.random.default_rng(6)
    x = rng.uniform(0, 1, (3, 10, 9))
    assert np.abs(OS.dssim_grad(x, x)).max() < 1e-12


def test_constant_planes_closed_form():
    """Constant planes x = a, y = b: at pixels >= 5 from every border the window sees
    no padding, the variances and covariance vanish and S reduces to the luminance
    term (2ab + C1) / (a^2 + b^2 + C1) -- [3DGS]'s SSIM with C2 / C2 = 1."""
    a, b = 0.7, 0.3
    x = np.full((1, 15, 17), a)
    y = np.full((1, 15, 17), b)
    S = OS.ssim_map(x, y)[0, 5:-5, 5:-5]
    want = (2 * a * b + OS.C1) / (a * a + b * b + OS.C1)
    np.testing.assert_allclose(S, want, rtol=1e-12)
