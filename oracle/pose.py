"""CPU oracle of N2's pose stage -- TEST INFRASTRUCTURE (see oracle/__init__.py
for who may import it).  numpy, float64, in the paper's order.

* Eq. 10: {R*, t*}, I* = argmin_{R,t} sum_i rho(||p_i - pi(K [R|t] g_i)||, tau)
  with SPEC's truncated quadratic rho(e, tau) = min(e^2, tau^2) and
  inliers e <= tau.  pi([x, y, z]) = [x/z, y/z], pixel =
  (fx x/z + cx, fy y/z + cy); a point with z <= 0 is an outlier.
* "PnP algorithm with RANSAC", reading Q35: the dense stage always
  starts from the pose it rendered at, so each RANSAC hypothesis is
  the exact fit of a minimal 3-correspondence sample by Gauss-Newton from
  that pose (6 residuals, 6 unknowns, NEWTON_ITERS steps); hypotheses are
  scored by inlier count (ties: lowest hypothesis index); the best is refined
  by damped Gauss-Newton on the truncated quadratic (inliers re-selected at
  every step, REFINE_ITERS steps).  Samples come from a counter-based hash
  (sample_index) that the GPU implements identically.
* Pose update: left perturbation xi = (v, w): R <- Exp(w) R, t <- Exp(w) t + v.
* Algorithm 2: Psi(T1, T2) = (arccos((clamp(tr(R1 R2^T), -1, 3) - 1) / 2)
  in degrees, |t1 - t2|); unreliable iff a consecutive pair exceeds tau = 20 deg
  (SPEC S:530 reads the loop as consecutive pairs).
"""
from __future__ import annotations

import math
from typing import Dict, List, Sequence

import numpy as np

TAU_PX = 3.0          # SPEC S:429 default
N_HYP = 128
NEWTON_ITERS = 8
REFINE_ITERS = 10
DAMPING = 1e-6        # relative Levenberg damping of the refinement normal equations
M32 = 0xFFFFFFFF


def sample_index(seed: int, h: int, k: int, n: int) -> int:
    """Counter-based hash (32-bit wrap-around arithmetic) -> index in [0, n)."""
    x = (seed * 0x9E3779B1 + h * 0x85EBCA77 + k * 0xC2B2AE3D) & M32
    x ^= x >> 16
    x = (x * 0x7FEB352D) & M32
    x ^= x >> 15
    x = (x * 0x846CA68B) & M32
    x ^= x >> 16
    return x % n


def minimal_sample(seed: int, h: int, n: int) -> List[int]:
    """Three distinct indices: draw k = 0, 1, 2, ...; skip repeats (at most 32 draws)."""
    out: List[int] = []
    k = 0
    while len(out) < 3 and k < 32:
        i = sample_index(seed, h, k, n)
        if i not in out:
            out.append(i)
        k += 1
    return out


def so3_exp(w: np.ndarray) -> np.ndarray:
    th = float(np.linalg.norm(w))
    Kx = np.array([[0, -w[2], w[1]], [w[2], 0, -w[0]], [-w[1], w[0], 0]], np.float64)
    if th < 1e-12:
        return np.eye(3) + Kx
    return np.eye(3) + math.sin(th) / th * Kx + (1 - math.cos(th)) / (th * th) * (Kx @ Kx)


def residuals(K, R, t, p2, X):
    """Reprojection residual [n][2] and camera depth z [n]."""
    fx, fy, cx, cy = K
    Pc = X @ R.T + t
    z = Pc[:, 2]
    zs = np.where(np.abs(z) > 1e-12, z, 1e-12)
    u = fx * Pc[:, 0] / zs + cx
    v = fy * Pc[:, 1] / zs + cy
    return np.stack([u - p2[:, 0], v - p2[:, 1]], 1), z, Pc


def jacobian(K, Pc):
    """d(pixel)/d(xi) for the left perturbation, [n][2][6]."""
    fx, fy = K[0], K[1]
    x, y, z = Pc[:, 0], Pc[:, 1], Pc[:, 2]
    n = len(z)
    du = np.zeros((n, 2, 3))
    du[:, 0, 0] = fx / z
    du[:, 0, 2] = -fx * x / (z * z)
    du[:, 1, 1] = fy / z
    du[:, 1, 2] = -fy * y / (z * z)
    A = np.zeros((n, 3, 6))
    A[:, :, :3] = np.eye(3)
    # d(Pc)/dw = -[Pc]x
    A[:, 0, 4], A[:, 0, 5] = z, -y
    A[:, 1, 3], A[:, 1, 5] = -z, x
    A[:, 2, 3], A[:, 2, 4] = y, -x
    return du @ A


def apply(R, t, xi):
    dR = so3_exp(xi[3:])
    return dR @ R, dR @ t + xi[:3]


def inliers(K, R, t, p2, X, tau):
    r, z, _ = residuals(K, R, t, p2, X)
    e = np.sqrt((r * r).sum(1))
    return (z > 0) & (e <= tau), e


def newton_minimal(K, R, t, p2, X):
    """Exact fit of 3 correspondences by Gauss-Newton from (R, t); None if singular."""
    for _ in range(NEWTON_ITERS):
        r, z, Pc = residuals(K, R, t, p2, X)
        if (z <= 0).any():
            return None
        J = jacobian(K, Pc).reshape(-1, 6)
        A = J.T @ J
        try:
            L = np.linalg.cholesky(A + 1e-12 * np.trace(A) / 6 * np.eye(6))
        except np.linalg.LinAlgError:
            return None
        xi = -np.linalg.solve(L.T, np.linalg.solve(L, J.T @ r.reshape(-1)))
        if not np.isfinite(xi).all():
            return None
        R, t = apply(R, t, xi)
    return R, t


def refine(K, R, t, p2, X, tau):
    """Damped Gauss-Newton on sum min(e^2, tau^2): inliers re-selected each step."""
    for _ in range(REFINE_ITERS):
        m, _ = inliers(K, R, t, p2, X, tau)
        if m.sum() < 3:
            break
        r, _, Pc = residuals(K, R, t, p2[m], X[m])
        J = jacobian(K, Pc).reshape(-1, 6)
        A = J.T @ J
        A = A + DAMPING * np.trace(A) / 6 * np.eye(6)
        xi = -np.linalg.solve(A, J.T @ r.reshape(-1))
        R, t = apply(R, t, xi)
    return R, t


def solve_pnp(K: Sequence[float], R0: np.ndarray, t0: np.ndarray, p2: np.ndarray, X: np.ndarray,
              tau: float = TAU_PX, n_hyp: int = N_HYP, seed: int = 0) -> Dict:
    """RANSAC (minimal 3-point Gauss-Newton hypotheses from the initial pose) +
    truncated-quadratic refinement.  p2 [n][2] pixels, X [n][3] world points."""
    K = np.asarray(K, np.float64)
    R0 = np.asarray(R0, np.float64).reshape(3, 3)
    t0 = np.asarray(t0, np.float64).reshape(3)
    p2 = np.asarray(p2, np.float64)
    X = np.asarray(X, np.float64)
    n = len(p2)
    best, best_h, best_cnt = (R0, t0), -1, inliers(K, R0, t0, p2, X, tau)[0].sum() if n else 0
    if n >= 3:
        for h in range(n_hyp):
            idx = minimal_sample(seed, h, n)
            if len(idx) < 3:
                continue
            fit = newton_minimal(K, R0, t0, p2[idx], X[idx])
            if fit is None:
                continue
            c = int(inliers(K, fit[0], fit[1], p2, X, tau)[0].sum())
            if c > best_cnt:
                best, best_h, best_cnt = fit, h, c
    R, t = refine(K, best[0], best[1], p2, X, tau) if n >= 3 else best
    m, e = inliers(K, R, t, p2, X, tau)
    return dict(R=R, t=t, inliers=m, n_inliers=int(m.sum()), mean_err=float(e[m].mean()) if m.any() else 0.0,
                best_hypothesis=best_h)


def pose_difference(R1, t1, R2, t2):
    """Algorithm 2's Psi: (angle in degrees, translation distance)."""
    tr = float(np.trace(np.asarray(R1) @ np.asarray(R2).T))
    tr = min(3.0, max(tr, -1.0))
    return math.degrees(math.acos((tr - 1.0) / 2.0)), float(np.linalg.norm(np.asarray(t1) - np.asarray(t2)))


def verify_consistency(poses: Sequence, tau_deg: float = 20.0):
    """('reliable', n - 1) or ('unreliable', i) for the first consecutive pair (i, i+1) over tau."""
    if len(poses) < 2:
        return "unreliable", -1
    for i in range(len(poses) - 1):
        th, _ = pose_difference(poses[i][0], poses[i][1], poses[i + 1][0], poses[i + 1][1])
        if th > tau_deg:
            return "unreliable", i
    return "reliable", len(poses) - 1
