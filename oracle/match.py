"""CPU oracle of the N2 row: coarse-to-fine probabilistic
mutual matching on rendered feature maps -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module; the product path never
does.  Plain numpy in float64, written in the paper's order:

* P:276 "we first perform matching on coarse query and rendered feature maps
  ... we set H_f/H_c = 8": coarse maps by w x w average pooling (reading Q31,
  SPEC S:517), w = 8.
* P:312-316 Eq. 11: M = cosine similarity (reading Q32: a zero feature vector
  has similarity 0), P_M = softmax_row(M/tau) (.) softmax_col(M/tau)
  (max-subtracted), then mutual nearest neighbours on P_M.
* MNN: (i, j) iff j is the row-i maximum of P_M, i the column-j
  maximum, and P_M[i, j] > p_min; equal maxima go to the lowest index
  (reading Q33; SPEC asks for a strict maximum -- the two differ only on exact
  ties).
* P:278 / P:316 fine stage: for each coarse match (i_c, j_c), Eq. 11 + MNN
  between the w x w fine pixels of query cell i_c and of rendered cell j_c
  (reading Q34), then a 3 x 3 soft-argmax of the window row of P around the
  MNN peak, clipped to the window ("sub-pixel level matching").
* P:278 "fully leverage the depth information": each fine match carries the
  rendered pixel's back-projected point (the integer peak's xyz/valid from
  gs_backproject, SPEC S:519 drops A < a_min through `valid`).

Defaults tau = 0.1, p_min = 0.05.
"""
from __future__ import annotations

from typing import Dict, Optional

import numpy as np

TAU = 0.1
P_MIN = 0.05
W = 8


def pool(F: np.ndarray, w: int = W) -> np.ndarray:
    """[D][H][W] -> [D][H/w][W/w] mean over w x w blocks (Q31)."""
    D, H, Wd = F.shape
    assert H % w == 0 and Wd % w == 0
    return F.astype(np.float64).reshape(D, H // w, w, Wd // w, w).mean(axis=(2, 4))


def normalize_rows(X: np.ndarray) -> np.ndarray:
    """Rows scaled to unit L2 norm; zero rows stay zero (Q32)."""
    X = X.astype(np.float64)
    n = np.sqrt((X * X).sum(axis=1, keepdims=True))
    return np.where(n > 0, X / np.where(n > 0, n, 1.0), 0.0)


def cosine(Q: np.ndarray, R: np.ndarray) -> np.ndarray:
    """M[i, j] = cos(q_i, r_j) for row-feature matrices [n][D]."""
    return normalize_rows(Q) @ normalize_rows(R).T


def pmm(M: np.ndarray, tau: float = TAU) -> np.ndarray:
    """Eq. 11: row softmax (.) column softmax of M / tau, max-subtracted."""
    S = M.astype(np.float64) / tau
    er = np.exp(S - S.max(axis=1, keepdims=True))
    row = er / er.sum(axis=1, keepdims=True)
    ec = np.exp(S - S.max(axis=0, keepdims=True))
    col = ec / ec.sum(axis=0, keepdims=True)
    return row * col


def mutual_nn(P: np.ndarray, p_min: float = P_MIN):
    """(row argmax, column argmax, match[i] = j or -1); argmax = first maximum (Q33)."""
    ra = P.argmax(axis=1)
    ca = P.argmax(axis=0)
    match = np.full(P.shape[0], -1, np.int64)
    for i in range(P.shape[0]):
        j = ra[i]
        if ca[j] == i and P[i, j] > p_min:
            match[i] = j
    return ra, ca, match


def cells(F: np.ndarray) -> np.ndarray:
    """[D][h][w] -> [h*w][D] (row-major cells)."""
    D = F.shape[0]
    return F.reshape(D, -1).T


def coarse_match(Fq: np.ndarray, Fr: np.ndarray, w: int = W, tau: float = TAU, p_min: float = P_MIN) -> Dict:
    """Coarse stage: pooled maps, cosine M (Hc Wc x Hc Wc), Eq. 11, MNN."""
    Q, R = cells(pool(Fq, w)), cells(pool(Fr, w))
    M = cosine(Q, R)
    P = pmm(M, tau)
    ra, ca, match = mutual_nn(P, p_min)
    prob = np.where(match >= 0, P[np.arange(len(match)), np.maximum(match, 0)], 0.0)
    return dict(M=M, P=P, row_arg=ra, col_arg=ca, match=match, prob=prob)


def window_pixels(cell: int, Wc: int, Wf: int, w: int = W) -> np.ndarray:
    """Flat fine-pixel indices of coarse cell `cell`, row-major inside the window."""
    cy, cx = divmod(cell, Wc)
    ys, xs = np.meshgrid(np.arange(cy * w, cy * w + w), np.arange(cx * w, cx * w + w), indexing="ij")
    return (ys * Wf + xs).reshape(-1)


def fine_match(Fq: np.ndarray, Fr: np.ndarray, coarse: np.ndarray, w: int = W, tau: float = TAU,
               p_min: float = P_MIN, xyz: Optional[np.ndarray] = None, valid: Optional[np.ndarray] = None) -> Dict:
    """Fine stage over every coarse match; dense per query fine pixel:
    peak (rendered flat pixel or -1), prob, refined rendered (x, y), xyz, valid."""
    D, H, Wf = Fq.shape
    Wc = Wf // w
    n = H * Wf
    peak = np.full(n, -1, np.int64)
    prob = np.zeros(n)
    ref = np.full((n, 2), np.nan)
    Xq, Xr = cells(Fq), cells(Fr)
    for ic, jc in enumerate(coarse):
        if jc < 0:
            continue
        qi = window_pixels(ic, Wc, Wf, w)
        rj = window_pixels(int(jc), Wc, Wf, w)
        P = pmm(cosine(Xq[qi], Xr[rj]), tau)
        _, _, m = mutual_nn(P, p_min)
        for a, b in enumerate(m):
            if b < 0:
                continue
            by, bx = divmod(int(b), w)
            num = np.zeros(2)
            den = 0.0
            for dy in (-1, 0, 1):
                for dx in (-1, 0, 1):
                    y, x = by + dy, bx + dx
                    if 0 <= y < w and 0 <= x < w:
                        p = P[a, y * w + x]
                        num += p * np.array([x, y], np.float64)
                        den += p
            cy, cx = divmod(int(jc), Wc)
            peak[qi[a]] = rj[b]
            prob[qi[a]] = P[a, b]
            ref[qi[a]] = [cx * w + num[0] / den, cy * w + num[1] / den]
    out = dict(peak=peak, prob=prob, ref=ref)
    if xyz is not None:
        pk = np.maximum(peak, 0)
        out["xyz"] = np.where(peak[:, None] >= 0, xyz.reshape(3, -1).T[pk], 0.0)
        out["valid"] = np.where(peak >= 0, valid.reshape(-1)[pk], 0).astype(np.uint8)
    return out
