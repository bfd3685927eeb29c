"""Small fixture builders shared by the tests (input construction only)."""
import json
import math
import os

import numpy as np

import synth

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
SH_C0 = 1.0 / (2.0 * math.sqrt(math.pi))  # Y_00 = 1/(2 sqrt(pi)) (textbook)


def golden(name):
    with open(os.path.join(GOLDEN, "fixtures.json")) as f:
        return json.load(f)[name]


def cam(d, R=None, t=None):
    return synth.make_view(np.eye(3) if R is None else R, np.zeros(3) if t is None else t,
                           d["fx"], d["fy"], d["cx"], d["cy"], d["width"], d["height"])


def scene_of(gs, sh_degree=0, feat=None):
    """gs: list of dicts with mu, scale (scalar or 3), quat (optional), opacity, rgb."""
    n = len(gs)
    pos = np.zeros((3, n), np.float32)
    quat = np.zeros((4, n), np.float32)
    scale = np.zeros((3, n), np.float32)
    op = np.zeros(n, np.float32)
    nk = (sh_degree + 1) ** 2
    sh = np.zeros((nk * 3, n), np.float32)
    for i, g in enumerate(gs):
        pos[:, i] = g["mu"]
        quat[:, i] = g.get("quat", [1.0, 0.0, 0.0, 0.0])
        s = g.get("scale", 0.1)
        scale[:, i] = s if np.ndim(s) else [s, s, s]
        op[i] = g.get("opacity", 0.99)
        rgb = np.asarray(g.get("rgb", [0.5, 0.5, 0.5]), np.float64)
        sh[0:3, i] = (rgb - 0.5) / SH_C0
        if "sh" in g:
            sh[:, i] = g["sh"]
    return synth.Scene(pos=pos, quat=quat, scale=scale, opacity=op, sh=sh, sh_degree=sh_degree,
                       feat=None if feat is None else np.asarray(feat, np.float32))


def random_tiny_scene(rng, n, feat_dim=0, sh_degree=0):
    """Random small scene in front of the 64x64 C1 camera, including edge cases:
    straddling the border, behind the camera, transparent, equal depths."""
    pos = np.stack([rng.uniform(-1.5, 1.5, n), rng.uniform(-1.5, 1.5, n), rng.uniform(-1, 8, n)])
    if n >= 4:
        pos[2, 1] = pos[2, 0]                    # exact depth tie -> gid tie-break
        pos[2, 3] = pos[2, 2]
    scale = np.exp(rng.uniform(math.log(0.01), math.log(0.5), (3, n)))
    q = rng.standard_normal((4, n)) * rng.uniform(0.5, 2.0, n)   # un-normalised quaternions
    op = rng.uniform(0.0, 1.0, n)
    nk = (sh_degree + 1) ** 2
    sh = rng.normal(0, 1.0, (nk * 3, n))
    feat = rng.standard_normal((n, feat_dim)).astype(np.float32) if feat_dim else None
    return synth.Scene(pos=pos.astype(np.float32), quat=q.astype(np.float32), scale=scale.astype(np.float32),
                       opacity=op.astype(np.float32), sh=sh.astype(np.float32), sh_degree=sh_degree, feat=feat)
