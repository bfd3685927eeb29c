"""Pins of the oracle's N2 row: coarse-to-fine probabilistic
mutual matching (Eq. 11).  Pins: the
hand-evaluated Eq. 11 values of SPEC S:468-469, softmax invariants, a
pure-Python MNN scan, the self-match and shift fixtures,
the 4096-fold search-space reduction and closed-form pooling."""
import math

import numpy as np
import pytest

from oracle import match as OM


def test_s468_singleton_softmax():
    for v in (-3.0, 0.0, 0.7):
        for tau in (0.01, 0.1, 2.0):
            assert OM.pmm(np.array([[v]]), tau)[0, 0] == pytest.approx(1.0, abs=1e-15)


def test_s469_identity_tau_one():
    """M = [[1,0],[0,1]], tau = 1 -> [[0.5344, 0.0723], [0.0723, 0.5344]],
    i.e. sigma(1)^2 and (1 - sigma(1))^2."""
    P = OM.pmm(np.eye(2), 1.0)
    s = math.e / (math.e + 1)
    np.testing.assert_allclose(P, [[s * s, (1 - s) ** 2], [(1 - s) ** 2, s * s]], rtol=1e-12)
    np.testing.assert_allclose(P, [[0.5344, 0.0723], [0.0723, 0.5344]], atol=5e-5)


@pytest.mark.parametrize("seed", range(5))
def test_eq11_invariants(seed):
    """Each factor is a softmax (rows resp. columns sum to 1); P <= min of the two
    factors; P(M^T) = P(M)^T; shifting M by a constant changes nothing."""
    rng = np.random.default_rng(seed)
    M = rng.uniform(-1, 1, (7, 9))
    tau = 0.1 + seed * 0.2
    P = OM.pmm(M, tau)
    e = np.exp(M / tau)
    row = e / e.sum(1, keepdims=True)
    col = e / e.sum(0, keepdims=True)
    np.testing.assert_allclose(row.sum(1), 1.0)
    np.testing.assert_allclose(col.sum(0), 1.0)
    assert (P <= np.minimum(row, col) + 1e-15).all()
    np.testing.assert_allclose(OM.pmm(M.T, tau), P.T, rtol=1e-12)
    np.testing.assert_allclose(OM.pmm(M + 0.37, tau), P, rtol=1e-12)


def test_small_tau_limit_is_mutual_indicator():
    """tau -> 0: P -> 1 exactly at mutual maxima, 0 elsewhere."""
    M = np.array([[0.9, 0.1, 0.2], [0.3, 0.8, 0.85], [0.0, 0.2, 0.1]])
    P = OM.pmm(M, 1e-3)
    # (0,0) is max of row 0 and column 0; (1,2) max of row 1 and column 2; row 2's max (col 1)
    # is not column 1's max (row 1)
    assert P[0, 0] > 0.999 and P[1, 2] > 0.999
    assert P[2].max() < 1e-6


def _mnn_scan(P, p_min):
    """The definition, as a plain double loop."""
    n, m = len(P), len(P[0])
    out = []
    for i in range(n):
        j = max(range(m), key=lambda c: (P[i][c], -c))
        col_best = max(range(n), key=lambda r: (P[r][j], -r))
        if col_best == i and P[i][j] > p_min:
            out.append((i, j))
    return out


@pytest.mark.parametrize("seed", range(6))
def test_mnn_equals_brute_force_scan(seed):
    """random 10x10 vs a brute-force MNN scan -> identical; one-to-one."""
    rng = np.random.default_rng(100 + seed)
    P = OM.pmm(rng.uniform(-1, 1, (10, 10)), 0.2)
    _, _, m = OM.mutual_nn(P, 0.0)
    got = [(i, int(j)) for i, j in enumerate(m) if j >= 0]
    assert got == _mnn_scan(P.tolist(), 0.0)
    js = [j for _, j in got]
    assert len(js) == len(set(js))


def test_mnn_row_max_not_column_max_excluded():
    P = np.array([[0.5, 0.4], [0.6, 0.1]])
    _, _, m = OM.mutual_nn(P, 0.0)
    assert m.tolist() == [-1, 0]          # row 0 -> col 0, but col 0's max is row 1


def test_pool_closed_form():
    F = np.arange(2 * 16 * 24, dtype=np.float64).reshape(2, 16, 24)
    Pm = OM.pool(F, 8)
    assert Pm.shape == (2, 2, 3)
    # mean of an arithmetic block = value at its centre: base + 3.5 rows * 24 + 3.5
    assert Pm[1, 1, 2] == pytest.approx(16 * 24 + (8 + 3.5) * 24 + 16 + 3.5)


def _feature_map(rng, D=16, H=64, Wd=64):
    # smooth-ish random field with distinct local structure
    F = rng.standard_normal((D, H, Wd))
    return F + 0.5 * np.roll(F, 1, axis=2) + 0.25 * np.roll(F, 1, axis=1)


def test_s486_self_match_diagonal_and_identical_pixels():
    rng = np.random.default_rng(7)
    F = _feature_map(rng)
    c = OM.coarse_match(F, F)
    assert (c["match"] == np.arange(len(c["match"]))).all()
    f = OM.fine_match(F, F, c["match"])
    n = F.shape[1] * F.shape[2]
    assert (f["peak"] == np.arange(n)).all()
    ys, xs = np.divmod(np.arange(n), F.shape[2])
    assert np.abs(f["ref"][:, 0] - xs).max() < 0.1 and np.abs(f["ref"][:, 1] - ys).max() < 0.1


def test_s487_shift_by_w_moves_coarse_matches_one_cell():
    rng = np.random.default_rng(8)
    F = _feature_map(rng)
    Fr = np.roll(F, 8, axis=2)                 # rendered = query shifted right by w = 8 px
    c = OM.coarse_match(F, Fr)
    Hc, Wc = F.shape[1] // 8, F.shape[2] // 8
    ok = 0
    for i, j in enumerate(c["match"]):
        cy, cx = divmod(i, Wc)
        if cx < Wc - 1:                        # the last column wraps around
            ok += int(j == cy * Wc + cx + 1)
    assert ok == Hc * (Wc - 1)


def test_s488_search_space_reduction():
    rng = np.random.default_rng(9)
    F = _feature_map(rng, D=4)
    c = OM.coarse_match(F, F)
    nf = F.shape[1] * F.shape[2]
    assert c["M"].shape == (nf // 64, nf // 64)
    assert (nf * nf) // c["M"].size == 4096


def test_fine_match_carries_backprojected_points():
    rng = np.random.default_rng(10)
    F = _feature_map(rng, D=8, H=32, Wd=32)
    xyz = rng.standard_normal((3, 32, 32))
    valid = (rng.uniform(size=(32, 32)) > 0.3).astype(np.uint8)
    c = OM.coarse_match(F, F)
    f = OM.fine_match(F, F, c["match"], xyz=xyz, valid=valid)
    np.testing.assert_array_equal(f["xyz"], xyz.reshape(3, -1).T)
    np.testing.assert_array_equal(f["valid"], valid.reshape(-1))
