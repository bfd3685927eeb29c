"""Pins of the oracle's N3 row: tight, opacity-aware binning
(reading Q30).  A record is binned only to the tiles of its 3-sigma rectangle
that the alpha >= alpha_min ellipse reaches.  The pins: the cut e_cut bounds
the exact threshold -log2(o / alpha_min) from below; the tile test never drops
a tile containing a pixel centre whose exact exponent reaches the cut (brute
force over the 256 centres, fp64); tight keys are a subset of square keys; and
the composited images and contributions are bit-identical in both modes."""
import math

import numpy as np
import pytest

import synth
from helpers import random_tiny_scene

K = -0.72134752044448170368   # reading Q29, k = -log2(e)/2


def test_e_cut_is_a_conservative_log2_threshold(orc):
    rng = np.random.default_rng(3)
    op = np.concatenate([rng.uniform(1 / 255, 1.0, 2000), [1 / 255, 1.0, 0.5, 2 / 255]]).astype(np.float32)
    sc = synth.box_v1(len(op), seed=5)
    sc.opacity[:] = op
    rec = orc.project(sc, synth.box_view())
    o = rec["opacity"].astype(np.float64)
    exact = -np.log2(o / np.float64(np.float32(1 / 255)))
    ec = rec["e_cut"].astype(np.float64)
    assert len(ec) > 100
    assert (ec <= exact * 1.05 - 0.0075 + 1e-6).all()            # at least the 5% + 0.0075 margin
    assert (ec >= exact * 1.05 - 0.0075 - 0.1).all()             # and not much more (log2 bound error < 0.09)


def _brute_force_hits(u, v, conic, ecut, tx, ty):
    """Any pixel centre of the tile with exact p(d) >= e_cut (fp64)."""
    ca, cb, cc = (float(x) for x in conic)
    xs = np.arange(16 * tx, 16 * tx + 16, dtype=np.float64)
    ys = np.arange(16 * ty, 16 * ty + 16, dtype=np.float64)
    dx = u - xs[None, :]
    dy = v - ys[:, None]
    p = K * 2.0 * (0.5 * (ca * dx * dx + cc * dy * dy) + cb * dx * dy)   # = -log2(e)/2 * q(d)
    return bool((p >= ecut + 1e-4).any())


@pytest.mark.parametrize("seed", range(6))
def test_tight_tiles_contain_every_reached_pixel(orc, seed):
    rng = np.random.default_rng(40 + seed)
    sc = random_tiny_scene(rng, 300)
    v = synth.make_view(np.eye(3), np.zeros(3), 60.0, 60.0, 47.5, 39.5, 96, 80)
    rec = orc.project(sc, v)
    sq = orc.bin_keys(rec, v, "square")
    ti = orc.bin_keys(rec, v, "tight")
    TX = (v.width + 15) // 16
    kept = set(zip(ti["tile"].tolist(), ti["rec"].tolist()))
    assert kept <= set(zip(sq["tile"].tolist(), sq["rec"].tolist()))
    dropped = 0
    for t, r in zip(sq["tile"].tolist(), sq["rec"].tolist()):
        if (t, r) in kept:
            continue
        dropped += 1
        assert not _brute_force_hits(float(rec["u"][r]), float(rec["v"][r]), rec["conic"][r],
                                     float(rec["e_cut"][r]), t % TX, t // TX), (t, r)
    assert dropped > 0


@pytest.mark.parametrize("cfg,scale", [("C1", 1.0), ("C2", 0.05), ("C4", 0.004)])
def test_tight_binning_renders_bit_identical_images(orc, cfg, scale):
    """The tiles tight binning drops contribute nothing: images, flags and
    per-record contributions are bit-identical to the square mode."""
    sc, vs = synth.make_config(cfg, scale=scale)
    v = vs[0]
    a = orc.render(sc, v, binning="square")
    b = orc.render(sc, v, binning="tight")
    assert len(b["keys"]["tile"]) < len(a["keys"]["tile"])
    for k in ("rgb", "depth", "alpha", "feat", "flags", "contrib"):
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)


def test_tight_binning_pair_reduction_on_nadir_aerial(orc):
    """C4 shape: the tight mode removes a large share of the 3-sigma square's pairs."""
    sc, vs = synth.make_config("C4", scale=0.01)
    rec = orc.project(sc, vs[0])
    n_sq = len(orc.bin_keys(rec, vs[0], "square")["tile"])
    n_ti = len(orc.bin_keys(rec, vs[0], "tight")["tile"])
    assert n_ti < 0.85 * n_sq, (n_ti, n_sq)
