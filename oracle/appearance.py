"""CPU oracle of Eq. 3's appearance-varied L1 term -- TEST INFRASTRUCTURE (see
oracle/__init__.py for who may import it).  numpy, float64.

P:146-150: L_rgb = (1 - lambda) (1/N) sum_i |I_i - I^a_i| + lambda L_D-SSIM(I, I^r),
with I^a the "appearance-varied rendered image" that "fits ground truth images
that may exhibit appearance variations relative to other images", while I^r
"achieves consistent appearance across views".  The paper (following
VastGaussian) does not give the appearance model.  Reading Q38: a
per-view, per-channel affine transform of the direct rendering,

    I^a_{v,c}(px) = a_{v,c} I^r_{v,c}(px) + b_{v,c},

trained jointly (identity init a = 1, b = 0) -- the simplest appearance variation
(exposure / white balance) that leaves I^r view-consistent.

appearance_l1(rendered, target, a, b, scale) with planes [P][H][W] (P = 3 x views,
plane p uses a[p], b[p]) returns (loss, dL/dI^r, dL/da, dL/db) of
L = scale sum |a I^r + b - I| (the subgradient sign(0) = 0).
"""
from __future__ import annotations

import numpy as np


def appearance_l1(rendered, target, a, b, scale: float):
    r = np.asarray(rendered, np.float64)
    t = np.asarray(target, np.float64)
    av = np.asarray(a, np.float64).reshape(-1, 1, 1)
    bv = np.asarray(b, np.float64).reshape(-1, 1, 1)
    d = av * r + bv - t
    s = np.sign(d)
    loss = scale * np.abs(d).sum()
    g_r = scale * s * av
    g_a = scale * (s * r).sum(axis=(1, 2))
    g_b = scale * s.sum(axis=(1, 2))
    return loss, g_r, g_a, g_b
