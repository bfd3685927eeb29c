"""CPU oracle of Eq. 3's D-SSIM term -- TEST INFRASTRUCTURE (see
oracle/__init__.py for who may import it).  numpy / scipy, float64.

P:146-150: L_rgb = (1 - lambda) L1 + lambda L_D-SSIM(I, I^r), the D-SSIM loss of
[3DGS] (Kerbl et al., cited there).  Reading Q37: D-SSIM = 1 - SSIM with SSIM the
mean over channels and pixels of

  S = ((2 mu_x mu_y + C1)(2 s_xy + C2)) / ((mu_x^2 + mu_y^2 + C1)(s_x^2 + s_y^2 + C2)),

local statistics under an 11 x 11 Gaussian window (sigma = 1.5, normalised),
zero padding ("same" size), C1 = 0.01^2, C2 = 0.03^2 -- [3DGS]'s constants.
"""
from __future__ import annotations

import numpy as np
from scipy.ndimage import correlate

C1, C2 = 0.01 ** 2, 0.03 ** 2


def window(size: int = 11, sigma: float = 1.5) -> np.ndarray:
    g = np.exp(-((np.arange(size) - size // 2) ** 2) / (2 * sigma * sigma))
    g /= g.sum()
    return np.outer(g, g)


def _blur(a, w):
    return correlate(a, w, mode="constant", cval=0.0)


def ssim_map(x, y) -> np.ndarray:
    """x, y: [C][H][W] -> S [C][H][W] (fp64)."""
    w = window()
    out = np.empty(np.shape(x))
    for c in range(np.shape(x)[0]):
        a, b = np.asarray(x[c], np.float64), np.asarray(y[c], np.float64)
        mx, my = _blur(a, w), _blur(b, w)
        sxx = _blur(a * a, w) - mx * mx
        syy = _blur(b * b, w) - my * my
        sxy = _blur(a * b, w) - mx * my
        out[c] = ((2 * mx * my + C1) * (2 * sxy + C2)) / ((mx * mx + my * my + C1) * (sxx + syy + C2))
    return out


def dssim(x, y) -> float:
    """Reading Q37: 1 - mean SSIM."""
    return float(1.0 - ssim_map(x, y).mean())


def dssim_grad(x, y) -> np.ndarray:
    """d dssim(x, y) / d x  [C][H][W] (fp64) -- the chain rule written out, for
    Eq. 3's D-SSIM gradient w.r.t. the rendered image I^r.  With
    A1 = 2 mu_x mu_y + C1, A2 = 2 s_xy + C2, B1 = mu_x^2 + mu_y^2 + C1,
    B2 = s_x^2 + s_y^2 + C2, S = A1 A2 / (B1 B2), and S a function of the window
    moments mu_x = w*x, E_xx = w*(x x), E_xy = w*(x y):
      dS/dmu_x = S (2 mu_y / A1 - 2 mu_y / A2 - 2 mu_x / B1 + 2 mu_x / B2)
      dS/dE_xx = -S / B2,   dS/dE_xy = 2 S / A2,
    and each moment is a zero-padded correlation with the symmetric window w,
    whose transpose is the same correlation:
      d sum_p S(p) / d x(q) = (w*dS/dmu_x)(q) + 2 x(q) (w*dS/dE_xx)(q) + y(q) (w*dS/dE_xy)(q).
    dssim = 1 - mean S, so the result is -1/(C H W) times that.  Pinned by central
    differences of dssim() in tests/test_ssim_oracle.py."""
    w = window()
    x = np.asarray(x, np.float64)
    y = np.asarray(y, np.float64)
    out = np.empty(x.shape)
    for c in range(x.shape[0]):
        a, b = x[c], y[c]
        mx, my = _blur(a, w), _blur(b, w)
        sxx = _blur(a * a, w) - mx * mx
        syy = _blur(b * b, w) - my * my
        sxy = _blur(a * b, w) - mx * my
        A1, A2 = 2 * mx * my + C1, 2 * sxy + C2
        B1, B2 = mx * mx + my * my + C1, sxx + syy + C2
        S = (A1 * A2) / (B1 * B2)
        d_mu = S * (2 * my / A1 - 2 * my / A2 - 2 * mx / B1 + 2 * mx / B2)
        d_xx = -S / B2
        d_xy = 2 * S / A2
        out[c] = _blur(d_mu, w) + 2 * a * _blur(d_xx, w) + b * _blur(d_xy, w)
    return -out / x.size
