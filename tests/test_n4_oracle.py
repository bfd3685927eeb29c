"""Pins of the oracle's N4 row: the feature-field backward of
Eq. 2 with the geometry frozen, dL/df_g = sum_px w_g(px) dL/dF(px).
Pins: exact linearity (a finite difference of the linear loss <g, F(f)> in f
equals the gradient to fp64 rounding), the sum identity sum_g dL/df_g = sum_px
A(px) g(px) (sum_k w_k = A), and binning-mode invariance."""
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
