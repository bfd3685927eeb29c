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
